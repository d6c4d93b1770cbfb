"""Blockwise 128 x 128 activation quantizer timing (tools only): bf16 at the DiT
(75600 x 5120 / 13824) and cfg2 (32760 x 1536 / 8960) shapes, CUDA events,
median of 20 (TB200_LIB selects a variant build)."""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_16093_b200 import ops  # noqa: E402

g = torch.Generator(device="cuda").manual_seed(0)
lib = os.path.basename(os.environ.get("TB200_LIB", "base"))
for (r, c) in ((75600, 5120), (32760, 1536), (32760, 8960), (75600, 13824)):
    x = torch.randn((r, c), generator=g, device="cuda").to(torch.bfloat16)
    for _ in range(3):
        ops.quantize_blockwise(x, 128, check_finite=False)
    ts = []
    for _ in range(20):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ops.quantize_blockwise(x, 128, check_finite=False)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = statistics.median(ts)
    print(f"{lib} {r}x{c}: {ms:.3f} ms, {3 * r * c / ms / 1e6:.0f} GB/s")
