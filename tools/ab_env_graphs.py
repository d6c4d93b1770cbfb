"""Same-process A/B/... of the cfg4 step under values of an environment knob read at
launch time by the library (tools only): one CUDA graph per value, replayed in
rotating order so box and drift effects cancel.  Usage: ab_env_graphs.py VAR v1 v2 ..."""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_16093_b200 import ops  # noqa: E402

H, L, D = 40, 75600, 128
g = torch.Generator(device="cuda").manual_seed(0)
q, k, v = (torch.randn((H, L, D), generator=g, device="cuda").to(torch.bfloat16) for _ in range(3))
var, vals = sys.argv[1], sys.argv[2:]


def capture(val):
    os.environ[var] = val
    for _ in range(2):
        ops.sla_attention(q, k, v, 128, 64, 0.1, 1.0, out_dtype=torch.bfloat16)
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        out = ops.sla_attention(q, k, v, 128, 64, 0.1, 1.0, out_dtype=torch.bfloat16)
    return gr, out


graphs = {val: capture(val) for val in vals}
for gr, _ in graphs.values():
    gr.replay()
torch.cuda.synchronize()
ref = graphs[vals[0]][1]
for val in vals[1:]:
    assert torch.equal(ref, graphs[val][1]), f"{var}={val} changes the output"
res = {val: [] for val in vals}
for rnd in range(10):
    order = vals[rnd % len(vals):] + vals[:rnd % len(vals)]
    for val in order:
        gr = graphs[val][0]
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            gr.replay()
        e1.record()
        torch.cuda.synchronize()
        res[val].append(e0.elapsed_time(e1) / 10)
for val in vals:
    print(f"{var}={val}: median {statistics.median(res[val]):.3f} ms  all {[round(x, 3) for x in res[val]]}")
