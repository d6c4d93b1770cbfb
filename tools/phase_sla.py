"""Whole-launch phase accounting of the fused kernel (trace build only):
average prologue / main-loop / epilogue cycles per CTA, per-SM busy span in
cycles and ns (-> effective SM clock), and the steady-state share.

    make -C paper_2512_16093_b200/csrc trace
    TB200_LIB=paper_2512_16093_b200/libtb200_trace.so python tools/phase_sla.py
"""
import ctypes
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_16093_b200 import _lib, ops  # noqa: E402

H, L, D = int(os.environ.get("TB_H", "40")), 75600, 128
g = torch.Generator(device="cuda").manual_seed(0)
q, k, v = (torch.randn((H, L, D), generator=g, device="cuda").to(torch.bfloat16) for _ in range(3))
_, parts = ops.sla_attention(q, k, v, 128, 64, 0.1, 1.0, out_dtype=torch.bfloat16, return_parts=True)
out = torch.empty((H, L, D), dtype=torch.bfloat16, device="cuda")
a = ops.sla_args(q=ops.ptr(q), k=ops.ptr(k), v=ops.ptr(v), dtype=1, H=H, L=L, d=D, q_block=128, kv_block=64,
                 count=parts["count"], scale=1.0 / math.sqrt(D), linear_mix=1.0, quantized=1,
                 q_codes=ops.ptr(parts["q_codes"]), k_codes=ops.ptr(parts["k_codes"]),
                 q_scales=ops.ptr(parts["q_scales"]), k_scales=ops.ptr(parts["k_scales"]),
                 k_mean=ops.ptr(parts["k_mean"]), idx=ops.ptr(parts["idx"]), vt=None, l_pad=-(-L // 64) * 64,
                 num_l=None, den_l=None, lin_ld=0, lin_hs=0, lin_kv=ops.ptr(parts["lin_kv"]),
                 lin_dx=parts["lin_kv"].shape[2], out=ops.ptr(out), out_dtype=1, row_max=None, den=None)
lib = _lib.load()
lib.tb_sla_phase_read.argtypes = [ctypes.c_void_p, ctypes.c_int]
buf = (ctypes.c_ulonglong * (4 + 160 * 4))()
for _ in range(3):
    lib.tb_sla_attention(ctypes.byref(a), ops.stream_ptr())
torch.cuda.synchronize()
lib.tb_sla_phase_read(ctypes.cast(buf, ctypes.c_void_p), 1)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
lib.tb_sla_attention(ctypes.byref(a), ops.stream_ptr())
e1.record()
torch.cuda.synchronize()
assert lib.tb_sla_phase_read(ctypes.cast(buf, ctypes.c_void_p), 1) == 0
b = np.array(buf, dtype=np.uint64)
ph = b[:4].astype(np.float64)
sm = b[4:].reshape(160, 4)[:148].astype(np.float64)
n = ph[3]
span_c = sm[:, 1] - sm[:, 0]
span_ns = sm[:, 3] - sm[:, 2]
count = parts["count"]
print(f"event time {e0.elapsed_time(e1):.3f} ms, CTAs {int(n)}")
print(f"per CTA: prologue {ph[0] / n:.0f}  main {ph[1] / n:.0f} ({ph[1] / n / count:.0f}/block)  epilogue {ph[2] / n:.0f} cycles")
print(f"per SM span: {span_c.mean() / 1e6:.3f} M cycles, {span_ns.mean() / 1e6:.3f} ms -> {span_c.mean() / span_ns.mean():.3f} GHz")
print(f"sum of CTA lifetimes / (2 x SM span): {(ph[0] + ph[1] + ph[2]) / (2 * span_c.sum()):.3f}")
print(f"main-loop share of CTA lifetime: {ph[1] / (ph[0] + ph[1] + ph[2]):.3f}")
units = H * (-(-L // 128)) * count
print(f"cycles per (q-tile, block) per SM: {span_c.mean() * 148 / units:.0f} (tensor floor ~464)")
