"""cfg4 step time (CUDA graph replay) for the prep-pass orderings of
ops.sla_attention (ops._PREP_ORDER: 0 = kv_part from t=0, 1 = after the Q pass,
2 = after the K pool), interleaved; tools only."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_16093_b200 import ops  # noqa: E402

H, L, D = 40, 75600, 128
g = torch.Generator(device="cuda").manual_seed(0)
q, k, v = (torch.randn((H, L, D), generator=g, device="cuda").to(torch.bfloat16) for _ in range(3))
ref = ops.sla_attention(q, k, v, 128, 64, 0.1, 1.0, out_dtype=torch.bfloat16)


def graph_ms(order):
    ops._PREP_ORDER = order
    fn = lambda: ops.sla_attention(q, k, v, 128, 64, 0.1, 1.0, out_dtype=torch.bfloat16)  # noqa: E731
    for _ in range(3):
        o = fn()
    torch.cuda.synchronize()
    assert torch.equal(o, ref), "ordering changed the result"
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


res = {o: [] for o in (0, 1, 2)}
for _ in range(3):
    for o in (0, 1, 2):
        res[o].append(graph_ms(o))
for o, t in res.items():
    print(f"order {o}: {[round(x, 3) for x in t]} ms, min {min(t):.3f}")
