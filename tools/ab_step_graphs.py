"""Same-process A/B of two variants of the cfg4 step (tools only): both are
captured as CUDA graphs and replayed alternately, so box-to-box and drift
effects cancel.  Variant toggles are module flags of ops (here: _KV_POOL)."""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_16093_b200 import ops  # noqa: E402

H, L, D = 40, 75600, 128
g = torch.Generator(device="cuda").manual_seed(0)
q, k, v = (torch.randn((H, L, D), generator=g, device="cuda").to(torch.bfloat16) for _ in range(3))
flag = sys.argv[1] if len(sys.argv) > 1 else "_KV_POOL"


def capture(val):
    setattr(ops, flag, val)
    for _ in range(2):
        ops.sla_attention(q, k, v, 128, 64, 0.1, 1.0, out_dtype=torch.bfloat16)
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        out = ops.sla_attention(q, k, v, 128, 64, 0.1, 1.0, out_dtype=torch.bfloat16)
    return gr, out


graphs = {True: capture(True), False: capture(False)}
for gr, _ in graphs.values():
    gr.replay()
torch.cuda.synchronize()
assert torch.equal(graphs[True][1], graphs[False][1]), "variants differ"
res = {True: [], False: []}
for rnd in range(8):
    for val in (True, False) if rnd % 2 == 0 else (False, True):
        gr = graphs[val][0]
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            gr.replay()
        e1.record()
        torch.cuda.synchronize()
        res[val].append(e0.elapsed_time(e1) / 10)
for val in (True, False):
    print(f"{flag}={val}: median {statistics.median(res[val]):.3f} ms  all {[round(x, 3) for x in res[val]]}")
