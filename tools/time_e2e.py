"""e2e (pinned host buffers -> device -> host) cfg4 SLA attention through
ops.sla_attention_host for several head-chunk sizes, plus the raw H2D / D2H
copy bandwidth of the same bytes (the PCIe bound)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_16093_b200 import ops  # noqa: E402

H, L, D = 40, 75600, 128
g = torch.Generator().manual_seed(0)
hq = [torch.randn((H, L, D), generator=g).to(torch.bfloat16).pin_memory() for _ in range(3)]
hout = torch.empty((H, L, D), dtype=torch.bfloat16).pin_memory()


def t(fn, n=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


dev = [torch.empty_like(x, device="cuda") for x in hq]
print(f"H2D 3 x {hq[0].numel() * 2 / 1e9:.2f} GB: {t(lambda: [d.copy_(h, non_blocking=True) for d, h in zip(dev, hq)]):.2f} ms")
print(f"D2H 1 x {hout.numel() * 2 / 1e9:.2f} GB: {t(lambda: hout.copy_(dev[0], non_blocking=True)):.2f} ms")
for ch in (1, 2, 4, 8):
    ms = t(lambda: ops.sla_attention_host(hq[0], hq[1], hq[2], 128, 64, 0.1, 1.0, out=hout, chunk_heads=ch))
    print(f"chunk_heads={ch}: {ms:.2f} ms", flush=True)
