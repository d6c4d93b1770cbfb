"""Time the fused SLA kernel alone at cfg4 (40 x 75600 x 128) for the library
selected by TB200_LIB; prints ms and TOPS (executed sparse work)."""
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
_, parts = ops.sla_attention(q, k, v, 128, 64, 0.1, 1.0, out_dtype=torch.bfloat16, return_parts=True)
l_pad = -(-L // 64) * 64
out = torch.empty((H, L, D), dtype=torch.bfloat16, device="cuda")
a = ops.sla_args(q=ops.ptr(q), k=ops.ptr(k), v=ops.ptr(v), dtype=1, H=H, L=L, d=D, q_block=128, kv_block=64,
                 count=parts["count"], scale=1.0 / math.sqrt(D), linear_mix=1.0, quantized=1,
                 q_codes=ops.ptr(parts["q_codes"]), k_codes=ops.ptr(parts["k_codes"]),
                 q_scales=ops.ptr(parts["q_scales"]), k_scales=ops.ptr(parts["k_scales"]),
                 k_mean=ops.ptr(parts["k_mean"]), idx=ops.ptr(parts["idx"]), vt=None, l_pad=l_pad,
                 num_l=None, den_l=None, lin_ld=0, lin_hs=0, lin_kv=ops.ptr(parts["lin_kv"]),
                 lin_dx=parts["lin_kv"].shape[2], out=ops.ptr(out), out_dtype=1, row_max=None, den=None)
FP8 = os.environ.get("TB_FP8", "0") == "1"      # opt-in FP8 P/V
if FP8:
    v8, v8s = ops.quant_v_fp8(v)
    a.v_fp8, a.v_scales = ops.ptr(v8), ops.ptr(v8s)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        ops.quant_v_fp8(v)
    e1.record()
    torch.cuda.synchronize()
    print(f"quant_v_fp8: {e0.elapsed_time(e1) / 10:.3f} ms")
lib = _lib.load()
for _ in range(3):
    lib.tb_sla_attention(ctypes.byref(a), ops.stream_ptr())
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    lib.tb_sla_attention(ctypes.byref(a), ops.stream_ptr())
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
ops_ = 4 * H * L * min(parts["count"] * 64, L) * D
print(f"{os.environ.get('TB200_LIB', 'libtb200.so')}{' fp8 P/V' if FP8 else ''}: {ms:.3f} ms  {ops_ / ms / 1e9:.1f} TOPS")
