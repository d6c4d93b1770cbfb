"""Wall time of the drop-in numpy call at cfg4 (tools only): attention.sla_attention
on numpy f32 [40, 75600, 128] inputs -> numpy f32, with the native host staging
(tb_host_stage) against torch's copy_, for a few head-chunk sizes."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2512_16093_b200 import attention, ops  # noqa: E402
from paper_2512_16093_b200.attention import AttnInputs, SLAConfig, sla_attention  # noqa: E402

H, L, D = 40, 75600, 128
g = torch.Generator(device="cuda").manual_seed(0)
x = [torch.randn((H, L, D), generator=g, device="cuda").to(torch.bfloat16).float().cpu().numpy() for _ in range(3)]
inp = AttnInputs(*x)
cfg = SLAConfig(q_block=128, kv_block=64, topk_ratio=0.1, linear_mix=1.0)
native = ops.host_stage
ref = None
for mode in ("native",):
    ops.host_stage = native if mode == "native" else (lambda d, s: d.copy_(s))
    for ch in (1, 2, 4):
        attention._HOST_CHUNK_HEADS = ch
        o = sla_attention(inp, cfg)
        if ref is None:
            ref = o.copy()
        assert np.array_equal(o, ref), "staging changed the result"
        del o
        ts = []
        for _ in range(4):
            t0 = time.perf_counter()
            o = sla_attention(inp, cfg)
            ts.append(time.perf_counter() - t0)
            del o
        print(f"drop-in e2e {mode} chunk {ch}: ms {[round(t * 1e3, 1) for t in ts]} median "
              f"{np.median(ts) * 1e3:.1f}", flush=True)
ops.host_stage = native
