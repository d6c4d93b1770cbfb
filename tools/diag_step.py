"""Diagnose the bench step (cfg4, 40 x 75600 x 128 bf16): per-step event times,
host launch time per step, a sync-debug pass, and a CUDA-graph replay."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_16093_b200 import ops  # noqa: E402

H, L, D = 40, 75600, 128
g = torch.Generator(device="cuda").manual_seed(0)
q, k, v = (torch.randn((H, L, D), generator=g, device="cuda").to(torch.bfloat16) for _ in range(3))


def step():
    return ops.sla_attention(q, k, v, 128, 64, 0.1, 1.0, out_dtype=torch.bfloat16)


for _ in range(3):
    step()
torch.cuda.synchronize()
torch.cuda.set_sync_debug_mode("warn")
step()
torch.cuda.set_sync_debug_mode(0)
torch.cuda.synchronize()

import bench  # noqa: E402

N = int(os.environ.get("DIAG_STEPS", "40"))
ev = [torch.cuda.Event(enable_timing=True) for _ in range(N + 1)]
host = []
with bench.ClockSampler(0) as clk:
    ev[0].record()
    for i in range(N):
        t0 = time.perf_counter()
        step()
        host.append((time.perf_counter() - t0) * 1e3)
        ev[i + 1].record()
    torch.cuda.synchronize()
print("per-step ms:", " ".join(f"{ev[i].elapsed_time(ev[i + 1]):.2f}" for i in range(N)))
print("host ms/step:", " ".join(f"{h:.2f}" for h in host))
print("mean ms:", ev[0].elapsed_time(ev[N]) / N)
print("clocks:", " ".join(f"{r[0]}/{r[2]}W{'P' if r[6] == 'Active' else ''}" for r in clk.rows))
print(clk.summary())

# graph replay
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    for _ in range(2):
        step()
torch.cuda.current_stream().wait_stream(s)
torch.cuda.synchronize()
try:
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        step()
    for _ in range(3):
        gr.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        gr.replay()
    e1.record()
    torch.cuda.synchronize()
    print("graph mean ms:", e0.elapsed_time(e1) / 10)
except Exception as e:  # noqa: BLE001
    print("graph capture failed:", repr(e))
