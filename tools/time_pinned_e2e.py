"""ops.sla_attention_host on pinned bf16 host tensors at cfg4 (tools only):
CUDA-event time per call with and without the single-head edge chunks."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_16093_b200 import ops  # noqa: E402

H, L, D = 40, 75600, 128
g = torch.Generator(device="cuda").manual_seed(0)
hq = [torch.randn((H, L, D), generator=g, device="cuda").to(torch.bfloat16).cpu().pin_memory() for _ in range(3)]
hout = torch.empty((H, L, D), dtype=torch.bfloat16).pin_memory()
for rep in range(2):
    for edge in (True, False):
        for ch in (4, 2):
            ops._HOST_EDGE_CHUNKS = edge
            ops.sla_attention_host(hq[0], hq[1], hq[2], 128, 64, 0.1, 1.0, out=hout, chunk_heads=ch)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(3):
                ops.sla_attention_host(hq[0], hq[1], hq[2], 128, 64, 0.1, 1.0, out=hout, chunk_heads=ch)
            e1.record()
            torch.cuda.synchronize()
            print(f"edge={int(edge)} chunk {ch}: {e0.elapsed_time(e1) / 3:.1f} ms", flush=True)
