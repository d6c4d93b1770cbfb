"""One cfg4 SLA step (BF16 P/V and FP8 P/V), one blockwise activation
quantization (75600 x 5120 bf16) and one W8A8 GEMM inside a
cudaProfilerStart/Stop region, for
  ncu --profile-from-start off --metrics <time, dram bytes, dram %, tensor %> python tools/prep_profile.py
(the per-kernel HBM / tensor-pipe table in profiles/)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_16093_b200 import ops  # noqa: E402

H, L, D = 40, 75600, 128
g = torch.Generator(device="cuda").manual_seed(0)
q, k, v = (torch.randn((H, L, D), generator=g, device="cuda").to(torch.bfloat16) for _ in range(3))
x = torch.randn((75600, 5120), generator=g, device="cuda").to(torch.bfloat16)
bt = torch.randint(-127, 128, (13824, 5120), dtype=torch.int8, device="cuda")
bs = torch.rand((40, 108), device="cuda") * 0.01


def work():
    ops.sla_attention(q, k, v, 128, 64, 0.1, 1.0, out_dtype=torch.bfloat16)
    ops.sla_attention(q, k, v, 128, 64, 0.1, 1.0, out_dtype=torch.bfloat16, pv_fp8=True)
    xq, xs = ops.quantize_blockwise(x, 128, check_finite=False)
    ops.w8a8_gemm(xq, xs, bt, bs, 128, None, torch.bfloat16, exact=False)


work()
torch.cuda.synchronize()
torch.cuda.profiler.start()
work()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
