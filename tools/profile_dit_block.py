"""One cfg5 DiT block (L 75600, dim 5120, 40 heads, FFN 13824) through
dit.block_forward, for a per-kernel launch list:

    ncu --metrics gpu__time_duration.sum --clock-control none -s <warm-up> --csv \\
        --log-file gpurun_out/dit_block.csv python tools/profile_dit_block.py

Without ncu it prints the CUDA-event time of the block (median of 5)."""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_16093_b200 import dit  # noqa: E402

L, DIM, H, FFN = 75600, 5120, 40, 13824
w = dit.random_layers(DIM, FFN, 1, seed=0)[0]
g = torch.Generator(device="cuda").manual_seed(1)
x = torch.randn((L, DIM), generator=g, device="cuda")
sla = dict(q_block=128, kv_block=64, topk_ratio=0.1, linear_mix=1.0)
pending = torch.randn((L, DIM), generator=g, device="cuda") * 0.01
reps = int(os.environ.get("DIT_REPS", "6"))
ts = []
for _ in range(reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    xi = x.clone()
    e0.record()
    dit.block_forward(xi, 1.0, w, H, sla, L, None, pending)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print(f"block_forward: median {statistics.median(ts[1:]):.2f} ms over {reps - 1} reps")
