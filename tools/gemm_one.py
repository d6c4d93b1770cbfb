import sys, torch
sys.path.insert(0, ".")
from paper_2512_16093_b200 import ops
M, K, N = 32760, 1536, 4608
xq = torch.randint(-127, 128, (M, K), dtype=torch.int8, device="cuda")
xs = torch.rand((-(-M // 128), K // 128), device="cuda") * 0.01
bt = torch.randint(-127, 128, (N, K), dtype=torch.int8, device="cuda")
bs = torch.rand((K // 128, N // 128), device="cuda") * 0.01
for _ in range(3):
    ops.w8a8_gemm(xq, xs, bt, bs, 128, out_dtype=torch.float32, exact=False)
torch.cuda.synchronize()
