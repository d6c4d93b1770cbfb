"""One W8A8 GEMM launch at a given shape (for ncu): python tools/gemm_one.py M K N [exact] [bf16]"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2512_16093_b200 import ops  # noqa: E402

M, K, N = (int(x) for x in sys.argv[1:4])
exact = len(sys.argv) > 4 and sys.argv[4] == "1"
od = torch.bfloat16 if len(sys.argv) > 5 and sys.argv[5] == "1" else torch.float32
xq = torch.randint(-127, 128, (M, K), dtype=torch.int8, device="cuda")
xs = torch.rand((-(-M // 128), K // 128), device="cuda") * 0.01
bt = torch.randint(-127, 128, (N, K), dtype=torch.int8, device="cuda")
bs = torch.rand((K // 128, N // 128), device="cuda") * 0.01
for _ in range(2):
    ops.w8a8_gemm(xq, xs, bt, bs, 128, out_dtype=od, exact=exact)
torch.cuda.synchronize()
