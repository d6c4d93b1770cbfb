"""Wall time of the drop-in numpy call at cfg4 (tools only): attention.sla_attention
on numpy f32 [40, 75600, 128] inputs -> numpy f32."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2512_16093_b200.attention import AttnInputs, SLAConfig, sla_attention  # noqa: E402

H, L, D = 40, 75600, 128
g = torch.Generator(device="cuda").manual_seed(0)
x = [torch.randn((H, L, D), generator=g, device="cuda").to(torch.bfloat16).float().cpu().numpy() for _ in range(3)]
inp = AttnInputs(*x)
cfg = SLAConfig(q_block=128, kv_block=64, topk_ratio=0.1, linear_mix=1.0)
sla_attention(inp, cfg)
ts = []
for _ in range(4):
    t0 = time.perf_counter()
    o = sla_attention(inp, cfg)
    ts.append(time.perf_counter() - t0)
print("drop-in e2e ms:", [round(t * 1e3, 1) for t in ts], "threads", torch.get_num_threads())
