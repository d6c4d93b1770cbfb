"""Per-block phase timeline of one sla_tc CTA (build with -DTB_SLA_TRACE)."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2512_16093_b200 import _lib, ops  # noqa: E402

H, L, D = 40, 75600, 128
g = torch.Generator(device="cuda").manual_seed(0)
q, k, v = (torch.randn((H, L, D), generator=g, device="cuda").to(torch.bfloat16) for _ in range(3))
for _ in range(2):
    ops.sla_attention(q, k, v, 128, 64, 0.1, 1.0, out_dtype=torch.bfloat16)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * (64 * 8))()
lib = _lib.load()
lib.tb_sla_trace_read.argtypes = [ctypes.c_void_p]
assert lib.tb_sla_trace_read(ctypes.cast(buf, ctypes.c_void_p)) == 0
t = np.array(buf, dtype=np.int64).reshape(64, 8)
t0 = t[0, 0]
names = ["wait_s", "s_ready", "max_done", "p_arrived", "ld_done", "exp_done", "st_done", "-"]
print("block " + " ".join(f"{n:>12s}" for n in names))
for j in range(40):
    print(f"{j:5d} " + " ".join(f"{int(x - t0):12d}" for x in t[j]))
d = np.diff(t[5:40, 3])
print("softmax period (cycles/block): median", np.median(d), "mean", d.mean())
print("softmax busy (s_ready -> p_arrived): median", np.median(t[5:40, 3] - t[5:40, 1]))
print("wait for S (wait_s -> s_ready): median", np.median(t[5:40, 1] - t[5:40, 0]))
print("S ready after P(j-1) arrival: median", np.median(t[6:40, 1] - t[5:39, 3]))
for a_, b_, nm in ((1, 4, "ldtm"), (4, 2, "max"), (2, 5, "exp"), (5, 6, "sttm"), (6, 3, "arrive")):
    print(f"phase {nm}: median {np.median(t[5:40, b_] - t[5:40, a_])}")
