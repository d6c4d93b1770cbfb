"""Host memory rates behind the drop-in numpy path (tools only): tb_host_stage
(native staging: copy and f32 -> bf16) vs torch copy_, alone and while a
pinned H2D DMA stream runs concurrently."""
import os
import sys
import threading
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_16093_b200 import _lib  # noqa: E402

lib = _lib.load()
print("host threads", lib.tb_host_threads(), "torch threads", torch.get_num_threads(), flush=True)
n = 155 * 1024 * 1024 // 4                       # one 4-head cfg4 f32 chunk of one tensor
x = np.random.default_rng(0).standard_normal(n, dtype=np.float32)
pin = torch.empty(n, dtype=torch.float32, pin_memory=True)
pb = torch.empty(n, dtype=torch.bfloat16, pin_memory=True)


def rate(fn, nbytes, reps=6):
    fn()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    return nbytes * reps / (time.perf_counter() - t0) / 1e9


xb = torch.from_numpy(x).to(torch.bfloat16).float().numpy()      # bf16-valued f32
cases = {
    "native copy f32": (lambda: lib.tb_host_stage(pin.data_ptr(), x.ctypes.data, n, 0, 0, 0), n * 4),
    "native f32->bf16 exact (bf16-valued)": (lambda: lib.tb_host_stage_bf16_exact(pb.data_ptr(), xb.ctypes.data, n, 0), n * 4),
    "native f32->bf16": (lambda: lib.tb_host_stage(pb.data_ptr(), x.ctypes.data, n, 0, 1, 0), n * 4),
    "torch copy_ f32": (lambda: pin.copy_(torch.from_numpy(x)), n * 4),
    "torch f32->bf16": (lambda: pb.copy_(torch.from_numpy(x)), n * 4),
}
for k, (fn, nb) in cases.items():
    print(f"{k}: {rate(fn, nb):.1f} GB/s (source bytes)", flush=True)

# concurrent pinned H2D stream (what the pipeline overlaps the staging with)
src = torch.empty(4 * n, dtype=torch.float32, pin_memory=True)
dev = torch.empty(4 * n, dtype=torch.float32, device="cuda")
s = torch.cuda.Stream()
torch.cuda.synchronize()
t0 = time.perf_counter()
with torch.cuda.stream(s):
    for _ in range(3):
        dev.copy_(src, non_blocking=True)
s.synchronize()
h2d_alone = 3 * 4 * n * 4 / (time.perf_counter() - t0) / 1e9
print(f"H2D pinned alone: {h2d_alone:.1f} GB/s", flush=True)
for k in ("native copy f32", "native f32->bf16", "native f32->bf16 exact (bf16-valued)", "torch copy_ f32"):
    fn, nb = cases[k]
    with torch.cuda.stream(s):
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record()
        for _ in range(3):
            dev.copy_(src, non_blocking=True)
        ev1.record()
    r = rate(fn, nb, reps=10)
    s.synchronize()
    print(f"{k} during H2D: {r:.1f} GB/s; H2D during it {3 * 4 * n * 4 / ev0.elapsed_time(ev1) / 1e6:.1f} GB/s",
          flush=True)
