"""cfg4 single-call pipeline (tb_sla_forward) step time, CUDA graph replay,
plus the K-codes pass alone (tools only; TB200_LIB selects a variant build)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_16093_b200 import ops  # noqa: E402

H, L, D = 40, 75600, 128
g = torch.Generator(device="cuda").manual_seed(0)
q, k, v = (torch.randn((H, L, D), generator=g, device="cuda").to(torch.bfloat16) for _ in range(3))
lib = ops._lib.load(require_device=True)
nbytes = int(lib.tb_sla_workspace_bytes(H, L, D, 128, 64, 0.1, 1.0, ops.TB_BF16))
ws = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
out = torch.empty((H, L, D), dtype=torch.bfloat16, device="cuda")


def step():
    ops.call("tb_sla_forward", ops.ptr(q), ops.ptr(k), ops.ptr(v), ops.TB_BF16, H, L, D, 128, 64, 0.1, 1.0,
             D ** -0.5, ops.ptr(ws), nbytes, ops.ptr(out), ops.TB_BF16, ops.stream_ptr())


def graph_ms(fn, reps=10, rounds=5):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        fn()
    for _ in range(3):
        gr.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(rounds):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            gr.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / reps)
    return sorted(ts)[len(ts) // 2]


km = ops.kmean(k)
kcodes = graph_ms(lambda: ops.pool_quant_tokens(k, 64, km, pool=False))
st = graph_ms(step)
ref = out.clone()
print(f"lib={os.path.basename(os.environ.get('TB200_LIB', 'base'))}: step {st:.3f} ms  K codes alone {kcodes:.3f} ms  "
      f"out_sum {out.float().abs().sum().item():.6e}")
