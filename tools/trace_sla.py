"""Per-block phase timeline of one sla_tc CTA (clock64, SM cycles).

Build the trace variant and run on the GPU box:
    make -C paper_2512_16093_b200/csrc trace      # -> paper_2512_16093_b200/libtb200_trace.so
    TB200_LIB=paper_2512_16093_b200/libtb200_trace.so python tools/trace_sla.py
"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_16093_b200 import _lib, ops  # noqa: E402

H, L, D = 40, 75600, 128
g = torch.Generator(device="cuda").manual_seed(0)
q, k, v = (torch.randn((H, L, D), generator=g, device="cuda").to(torch.bfloat16) for _ in range(3))
for _ in range(2):
    ops.sla_attention(q, k, v, 128, 64, 0.1, 1.0, out_dtype=torch.bfloat16)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * (80 * 16))()
lib = _lib.load()
lib.tb_sla_trace_read.argtypes = [ctypes.c_void_p]
assert lib.tb_sla_trace_read(ctypes.cast(buf, ctypes.c_void_p)) == 0
t = np.array(buf, dtype=np.int64).reshape(80, 16)
t0 = t[0, 10]
names = {10: "tma_k", 11: "tma_v", 15: "qk_wait", 8: "mma_qk", 0: "sm_wait", 1: "s_ready", 4: "ld_done",
         5: "exp_done", 6: "st_done", 3: "p_arr0", 12: "p_arr3", 13: "pv_wait", 14: "v_ok", 9: "mma_pv"}
cols = [10, 11, 15, 8, 0, 1, 4, 5, 6, 3, 12, 13, 14, 9]
print("block " + " ".join(f"{names[c]:>9s}" for c in cols))
for j in range(48):
    print(f"{j:5d} " + " ".join(f"{int(t[j, c] - t0):9d}" for c in cols))
sl = slice(8, 40)
med = lambda a, b: float(np.median(t[sl, b] - t[sl, a]))
print("period (p_arr0 j -> j+1):", float(np.median(np.diff(t[8:41, 3]))))
print("softmax: wait S", med(0, 1), " ldtm", med(1, 4), " exp", med(4, 5), " sttm", med(5, 6), " arrive", med(6, 3))
print("S ready after P(j-1) arrival:", float(np.median(t[9:41, 1] - t[8:40, 3])))
print("PV(j) issue after P(j) arrival:", med(3, 9), "  warp-3 arrival lag:", med(3, 12))
print("QK(j) issue -> S(j) seen by softmax:", float(np.median(t[sl, 1] - t[sl, 8])))
p = t[70, :9] - t[70, 0]
print("prologue (from entry): setup barrier", p[1], " k1 wait start", p[2], " k1 ready", p[3], " phi stored", p[4], " phiq arrive", p[5], " corr+phi done", p[6], " c1 table", p[7], " named bar", p[8], " | tma_k(0)", t0 - t[70, 0], " s_ready(0)", t[0, 1] - t[70, 0])
e = t[71, :5] - t[71, 0]
print("epilogue: o_final wait", e[1], " phi(Q) done", e[2], " lin MMA done", e[3], " stores done", e[4])
print("QK(j+1) issue after PV(j-1) issue:", float(np.median(t[9:41, 8] - t[7:39, 9])))
