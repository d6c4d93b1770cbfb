"""Graph-mode timeline of the cfg4 step (tools only): ops.sla_attention's prep
passes re-issued with tb_timestamp kernels (%globaltimer) after each pass on
its stream, captured in a CUDA graph like bench.py's step, replayed; prints
the median end time of every pass relative to the step start.
Usage: python tools/step_timeline.py [order ...]: 3 = the shipped order (kv_part pools K),
0-2 = the earlier orders with a separate K pooling pass."""
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_16093_b200 import _lib, ops  # noqa: E402

H, L, D = 40, 75600, 128
g = torch.Generator(device="cuda").manual_seed(0)
q, k, v = (torch.randn((H, L, D), generator=g, device="cuda").to(torch.bfloat16) for _ in range(3))
nkv = -(-L // 64)
count = ops.topk_count(0.1, nkv)
lib = _lib.load()
ts = torch.zeros(32, dtype=torch.int64, device="cuda")
names = []


def stamp(name, stream=None):
    s = stream or torch.cuda.current_stream()
    if name not in names:
        names.append(name)
    lib.tb_timestamp(ts.data_ptr() + 8 * names.index(name), s.cuda_stream)


side, third = torch.cuda.Stream(), torch.cuda.Stream()


def step(order):
    main = torch.cuda.current_stream()
    stamp("start", main)
    side.wait_stream(main)
    with torch.cuda.stream(side):
        km = ops.kmean(k)
        stamp("k_mean", side)
        if order == 0:
            kc, ks, _ = ops.pool_quant_tokens(k, 64, km, pool=False)
            stamp("K codes", side)
    if order in (0, 3, 4):
        third.wait_stream(main)
    if order == 3:                     # kv_part pools the raw K blocks itself
        with torch.cuda.stream(third):
            kv_part, kp, kpt = ops.linear_kv_part(k, v, 64, pool=True)
            stamp("kv_part + K pool", third)
    qc, qs, qp = ops.pool_quant_tokens(q, 128, None, pool=True)
    stamp("Q pass", main)
    if order == 4:                     # the same, kv_part enqueued after the Q pass
        with torch.cuda.stream(third):
            kv_part, kp, kpt = ops.linear_kv_part(k, v, 64, pool=True)
            stamp("kv_part + K pool", third)
    if order in (3, 4):
        main.wait_stream(third)
    else:
        if order == 1:
            third.wait_stream(main)
        kp, kpt = ops.pool_tokens_t(k, 64)
        stamp("K pool", main)
        if order == 2:
            third.wait_stream(main)
        with torch.cuda.stream(third):
            kv_part = ops.linear_kv_part(k, v, 64)
            stamp("kv_part", third)
    idx, comp, cov = ops.topk_blocks_cov(qp, kp, count, want_comp=False, kpt=kpt)
    stamp("top-k", main)
    if order != 0:
        side.wait_stream(main)
        with torch.cuda.stream(side):
            kc, ks, _ = ops.pool_quant_tokens(k, 64, km, pool=False)
            stamp("K codes", side)
    main.wait_stream(third)
    lin_kv = ops.linear_kv_sel(kv_part, cov, nkv)
    stamp("coverage GEMM", main)
    main.wait_stream(side)
    out = torch.empty((H, L, D), dtype=torch.bfloat16, device="cuda")
    a = ops.sla_args(q=ops.ptr(q), k=ops.ptr(k), v=ops.ptr(v), dtype=1, H=H, L=L, d=D, q_block=128, kv_block=64,
                     count=count, scale=1.0 / math.sqrt(D), linear_mix=1.0, quantized=1, q_codes=ops.ptr(qc),
                     k_codes=ops.ptr(kc), q_scales=ops.ptr(qs), k_scales=ops.ptr(ks), k_mean=ops.ptr(km),
                     idx=ops.ptr(idx), vt=None, l_pad=nkv * 64, num_l=None, den_l=None, lin_ld=0, lin_hs=0,
                     lin_kv=ops.ptr(lin_kv), lin_dx=lin_kv.shape[2], out=ops.ptr(out), out_dtype=1,
                     row_max=None, den=None)
    import ctypes
    lib.tb_sla_attention(ctypes.byref(a), main.cuda_stream)
    stamp("fused kernel", main)
    for t in (km, kc, ks, kv_part):
        t.record_stream(main)
    return out


for order in [int(x) for x in sys.argv[1:]] or [3, 4, 0]:
    for _ in range(2):
        step(order)
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        step(order)
    runs = []
    for _ in range(7):
        gr.replay()
        torch.cuda.synchronize()
        t = ts.cpu().tolist()
        runs.append({n: (t[i] - t[0]) / 1e6 for i, n in enumerate(names)})
    print(f"order {order}: graph replay, ms from the step start (median of 7)")
    for n in sorted(names, key=lambda n: sorted(r[n] for r in runs)[3]):
        print(f"  {sorted(r[n] for r in runs)[3]:7.3f}  {n}")
