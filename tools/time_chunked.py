"""Head-chunked SLA step at cfg4: the prep passes of head chunk c+1 (on one
stream) overlap the fused kernel of chunk c (on another).  Times the plain
step and chunked variants, eager and CUDA-graph replayed."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_16093_b200 import ops  # noqa: E402

H, L, D = 40, 75600, 128
g = torch.Generator(device="cuda").manual_seed(0)
q, k, v = (torch.randn((H, L, D), generator=g, device="cuda").to(torch.bfloat16) for _ in range(3))
out = torch.empty((H, L, D), dtype=torch.bfloat16, device="cuda")
prio = int(os.environ.get("TB_PRIO", "0"))
lo, hi = torch.cuda.Stream.priority_range() if hasattr(torch.cuda.Stream, "priority_range") else (0, -1)
streams = [torch.cuda.Stream(priority=hi if prio else 0) for _ in range(2)]


def plain():
    ops.sla_attention(q, k, v, 128, 64, 0.1, 1.0, out_dtype=torch.bfloat16)


def chunked(nc):
    hs = [round(i * H / nc) for i in range(nc + 1)]
    main = torch.cuda.current_stream()
    for s in streams:
        s.wait_stream(main)
    for c in range(nc):
        s = streams[c % 2]
        with torch.cuda.stream(s):
            o = ops.sla_attention(q[hs[c]:hs[c + 1]], k[hs[c]:hs[c + 1]], v[hs[c]:hs[c + 1]], 128, 64, 0.1, 1.0,
                                  out_dtype=torch.bfloat16)
            out[hs[c]:hs[c + 1]].copy_(o) if False else None
    for s in streams:
        main.wait_stream(s)


def timeit(fn, graph):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    if graph:
        cap = torch.cuda.Stream()
        cap.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(cap):
            fn()
        torch.cuda.current_stream().wait_stream(cap)
        torch.cuda.synchronize()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr):
            fn()
        run = gr.replay
    else:
        run = fn
    for _ in range(2):
        run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        run()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 10


for graph in (False, True):
    print(f"graph={graph} plain: {timeit(plain, graph):.3f} ms", flush=True)
    for nc in (2, 4, 5, 8):
        print(f"graph={graph} chunks={nc}: {timeit(lambda: chunked(nc), graph):.3f} ms", flush=True)
