"""Where the cfg4 step's prep time goes (tools only): CUDA-graph timings of the
full ops.sla_attention step, the fused kernel alone, and subsets of the prep
passes on their streams (same calls as ops.sla_attention's fast path)."""
import ctypes
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_16093_b200 import _lib, ops  # noqa: E402

H, L, D = int(os.environ.get("TB_H", "40")), 75600, 128
g = torch.Generator(device="cuda").manual_seed(0)
q, k, v = (torch.randn((H, L, D), generator=g, device="cuda").to(torch.bfloat16) for _ in range(3))
nkv = -(-L // 64)
count = ops.topk_count(0.1, nkv)
_, parts = ops.sla_attention(q, k, v, 128, 64, 0.1, 1.0, out_dtype=torch.bfloat16, return_parts=True)
lib = _lib.load()
out = torch.empty((H, L, D), dtype=torch.bfloat16, device="cuda")
a = ops.sla_args(q=ops.ptr(q), k=ops.ptr(k), v=ops.ptr(v), dtype=1, H=H, L=L, d=D, q_block=128, kv_block=64,
                 count=count, scale=1.0 / math.sqrt(D), linear_mix=1.0, quantized=1,
                 q_codes=ops.ptr(parts["q_codes"]), k_codes=ops.ptr(parts["k_codes"]),
                 q_scales=ops.ptr(parts["q_scales"]), k_scales=ops.ptr(parts["k_scales"]),
                 k_mean=ops.ptr(parts["k_mean"]), idx=ops.ptr(parts["idx"]), vt=None, l_pad=nkv * 64,
                 num_l=None, den_l=None, lin_ld=0, lin_hs=0, lin_kv=ops.ptr(parts["lin_kv"]),
                 lin_dx=parts["lin_kv"].shape[2], out=ops.ptr(out), out_dtype=1, row_max=None, den=None)
main = torch.cuda.current_stream()
side, third = torch.cuda.Stream(), torch.cuda.Stream()


def prep(main_chain=True, cov=True, sidek=True, kvpart=True):
    main = torch.cuda.current_stream()
    side.wait_stream(main)
    third.wait_stream(main)
    kv_part = None
    if kvpart:
        with torch.cuda.stream(third):
            kv_part = ops.linear_kv_part(k, v, 64)
    if sidek:
        with torch.cuda.stream(side):
            km = ops.kmean(k)
            ops.pool_quant_tokens(k, 64, km, pool=False)
    if main_chain:
        qc, qs, qp = ops.pool_quant_tokens(q, 128, None, pool=True)
        kp, kpt = ops.pool_tokens_t(k, 64)
        idx, comp, cv = ops.topk_blocks_cov(qp, kp, count, want_comp=False, kpt=kpt)
        main.wait_stream(third)
        if cov and kv_part is not None:
            ops.linear_kv_sel(kv_part, cv, nkv)
    main.wait_stream(side)
    main.wait_stream(third)


def fused():
    lib.tb_sla_attention(ctypes.byref(a), ops.stream_ptr())


cases = {
    "full step (ops.sla_attention)": lambda: ops.sla_attention(q, k, v, 128, 64, 0.1, 1.0, out_dtype=torch.bfloat16),
    "fused kernel alone": fused,
    "prep, all passes": lambda: prep(),
    "prep without the coverage GEMM": lambda: prep(cov=False),
    "prep, main chain only (Q pass, K pool, top-k, coverage GEMM; kv_part too)": lambda: prep(sidek=False),
    "prep, side chains only (k_mean + K codes, kv_part)": lambda: prep(main_chain=False),
    "prep, k_mean + K codes only": lambda: prep(main_chain=False, kvpart=False),
    "prep + fused": lambda: (prep(), fused()),
}


def timeit(fn):
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
    for _ in range(10):
        gr.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 10


for name, fn in cases.items():
    print(f"{timeit(fn):8.3f} ms  {name}", flush=True)


# ---- timeline of one eager prep (CUDA events around every pass, per stream)
def timeline():
    main = torch.cuda.current_stream()
    ev = {}

    def mark(name, s):
        e = torch.cuda.Event(enable_timing=True)
        e.record(s)
        ev[name] = e

    mark("t0", main)
    side.wait_stream(main)
    third.wait_stream(main)
    with torch.cuda.stream(third):
        kv_part = ops.linear_kv_part(k, v, 64)
        mark("kv_part end", third)
    with torch.cuda.stream(side):
        km = ops.kmean(k)
        mark("k_mean end", side)
        ops.pool_quant_tokens(k, 64, km, pool=False)
        mark("K codes end", side)
    qc, qs, qp = ops.pool_quant_tokens(q, 128, None, pool=True)
    mark("Q pass end", main)
    kp, kpt = ops.pool_tokens_t(k, 64)
    mark("K pool end", main)
    idx, comp, cv = ops.topk_blocks_cov(qp, kp, count, want_comp=False, kpt=kpt)
    mark("top-k end", main)
    main.wait_stream(third)
    mark("kv_part joined", main)
    ops.linear_kv_sel(kv_part, cv, nkv)
    mark("coverage GEMM end", main)
    main.wait_stream(side)
    fused()
    mark("fused end", main)
    torch.cuda.synchronize()
    return {n: ev["t0"].elapsed_time(e) for n, e in ev.items() if n != "t0"}


for _ in range(3):
    timeline()
res = [timeline() for _ in range(5)]
print("eager timeline, ms from the start (median of 5):")
for n in res[0]:
    vals = sorted(r[n] for r in res)
    print(f"  {vals[2]:7.3f}  {n}")
