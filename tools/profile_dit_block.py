"""Per-op CUDA-event breakdown of one cfg5 DiT block (L 75600, dim 5120, 40 heads, FFN 13824)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_16093_b200 import dit, ops  # noqa: E402

L, DIM, H, FFN = 75600, 5120, 40, 13824
w = dit.random_layers(DIM, FFN, 1, seed=0)[0]
g = torch.Generator(device="cuda").manual_seed(1)
x = torch.randn((L, DIM), generator=g, device="cuda")
sla = dict(q_block=128, kv_block=64, topk_ratio=0.1, linear_mix=1.0)
times = {}


def timed(name, fn):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    r = fn()
    e1.record()
    torch.cuda.synchronize()
    times[name] = times.get(name, 0.0) + e0.elapsed_time(e1)
    return r


for it in range(4):
    times.clear()
    hd = DIM // H
    x1 = timed("emb add", lambda: x + 0.5 * w.sigma_emb)
    a = timed("rmsnorm", lambda: ops.rmsnorm(x1, w.rms_gain))
    aq = timed("act quant qkv", lambda: ops.quantize_blockwise(a, 128, check_finite=False))
    qkv = timed("gemm qkv", lambda: ops.w8a8_gemm(aq[0], aq[1], w.qkv.bt, w.qkv.scales, 128, None, torch.bfloat16, False))
    q, k, v = (t.view(L, H, hd) for t in qkv.split(DIM, dim=1))
    qh, kh, vh = timed("permute qkv", lambda: [t.permute(1, 0, 2).contiguous() for t in (q, k, v)])
    o = timed("sla attention", lambda: ops.sla_attention(qh, kh, vh, 128, 64, 0.1, 1.0, True, out_dtype=torch.bfloat16))
    o2 = timed("permute o", lambda: o.permute(1, 0, 2).reshape(L, DIM).contiguous())
    oq = timed("act quant out", lambda: ops.quantize_blockwise(o2, 128, check_finite=False))
    po = timed("gemm out", lambda: ops.w8a8_gemm(oq[0], oq[1], w.out_proj.bt, w.out_proj.scales, 128, None, torch.float32, False))
    x2 = timed("residual 1", lambda: x1 + po)
    b = timed("layernorm", lambda: ops.layernorm(x2, w.ln_gain, w.ln_offset))
    bq = timed("act quant mlp_in", lambda: ops.quantize_blockwise(b, 128, check_finite=False))
    h1 = timed("gemm mlp_in", lambda: ops.w8a8_gemm(bq[0], bq[1], w.mlp_in.bt, w.mlp_in.scales, 128, None, torch.bfloat16, False))
    h2 = timed("gelu", lambda: torch.nn.functional.gelu(h1, approximate="tanh"))
    hq = timed("act quant mlp_out", lambda: ops.quantize_blockwise(h2, 128, check_finite=False))
    p2 = timed("gemm mlp_out", lambda: ops.w8a8_gemm(hq[0], hq[1], w.mlp_out.bt, w.mlp_out.scales, 128, None, torch.float32, False))
    x3 = timed("residual 2", lambda: x2 + p2)
tot = sum(times.values())
for k_, v_ in times.items():
    print(f"{k_:20s} {v_:8.3f} ms  {100 * v_ / tot:5.1f}%")
print(f"{'total':20s} {tot:8.3f} ms")
