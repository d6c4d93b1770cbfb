"""k_mean alone and beside kv_part + the Q pass (the step's first prep phase) at cfg4; tools only.
Prints the k_mean stream's elapsed time in both settings (median of 7)."""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_16093_b200 import ops  # noqa: E402

H, L, D = 40, 75600, 128
g = torch.Generator(device="cuda").manual_seed(0)
q, k, v = (torch.randn((H, L, D), generator=g, device="cuda").to(torch.bfloat16) for _ in range(3))
sa, sb, sc = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()


def run(contended):
    torch.cuda.synchronize()
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    cur = torch.cuda.current_stream()
    e0.record(cur)
    for s in (sa, sb, sc):
        s.wait_event(e0)
    with torch.cuda.stream(sa):
        ops.kmean(k)
        e1.record(sa)
    if contended:
        with torch.cuda.stream(sb):
            ops.linear_kv_part(k, v, 64, pool=True)
        with torch.cuda.stream(sc):
            ops.pool_quant_tokens(q, 128, None, pool=True)
    for s in (sb, sc):
        e2.record(s)
        cur.wait_event(e2)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


for c in (False, True):
    for _ in range(3):
        run(c)
    t = statistics.median(run(c) for _ in range(7))
    print(f"{os.environ.get('TB200_LIB', 'libtb200.so').split('/')[-1]} k_mean {'beside kv_part + Q pass' if c else 'alone'}: {t:.3f} ms")
