"""W8A8 GEMM microbenchmark on the cfg2 sweep and the cfg5 DiT projection shapes."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2512_16093_b200 import ops  # noqa: E402

SHAPES = [(32760, 1536, 1536), (32760, 1536, 4608), (32760, 1536, 8960), (32760, 8960, 1536),
          (75600, 5120, 15360), (75600, 5120, 5120), (75600, 5120, 13824), (75600, 13824, 5120)]


def run(M, K, N, exact, out_dtype, reps=5):
    xq = torch.randint(-127, 128, (M, K), dtype=torch.int8, device="cuda")
    xs = torch.rand((-(-M // 128), K // 128), device="cuda") * 0.01
    bt = torch.randint(-127, 128, (N, K), dtype=torch.int8, device="cuda")
    bs = torch.rand((K // 128, N // 128), device="cuda") * 0.01
    for _ in range(2):
        ops.w8a8_gemm(xq, xs, bt, bs, 128, out_dtype=out_dtype, exact=exact)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        ops.w8a8_gemm(xq, xs, bt, bs, 128, out_dtype=out_dtype, exact=exact)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    return ms, 2 * M * K * N / (ms * 1e-3) / 1e12


if __name__ == "__main__":
    only = sys.argv[1] if len(sys.argv) > 1 else None
    for (M, K, N) in SHAPES:
        if only and only != f"{M}x{K}x{N}":
            continue
        for exact, od in ((True, torch.float32), (False, torch.float32), (False, torch.bfloat16)):
            ms, tops = run(M, K, N, exact, od)
            print(json.dumps({"M": M, "K": K, "N": N, "exact": exact, "out": str(od), "ms": round(ms, 4),
                              "TOPS": round(tops, 1)}), flush=True)
