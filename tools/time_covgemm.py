"""cfg4 coverage GEMM (cov . kv_part, 40 heads) alone and the full step, CUDA
graph replay (tools only)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_16093_b200 import ops  # noqa: E402

H, L, D = 40, 75600, 128
g = torch.Generator(device="cuda").manual_seed(0)
q, k, v = (torch.randn((H, L, D), generator=g, device="cuda").to(torch.bfloat16) for _ in range(3))
nkv = -(-L // 64)
count = ops.topk_count(0.1, nkv)
_, _, qp = ops.pool_quant_tokens(q, 128, None, pool=True)
kp, kpt = ops.pool_tokens_t(k, 64)
idx, comp, cov = ops.topk_blocks_cov(qp, kp, count, want_comp=False, kpt=kpt)
kv_part = ops.linear_kv_part(k, v, 64)


def graph_ms(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        fn()
    for _ in range(3):
        gr.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        gr.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


gemm = graph_ms(lambda: ops.linear_kv_sel(kv_part, cov, nkv))
step = graph_ms(lambda: ops.sla_attention(q, k, v, 128, 64, 0.1, 1.0, out_dtype=torch.bfloat16))
print(f"T2={os.environ.get('TB_GEMM_T2', '1')} coverage GEMM {gemm:.3f} ms ({0.9296e3 / gemm:.0f} TFLOP/s), "
      f"step {step:.3f} ms")
