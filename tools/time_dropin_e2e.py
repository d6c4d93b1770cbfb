"""Wall time of the drop-in numpy call at cfg4 (tools only): attention.sla_attention
on numpy f32 [40, 75600, 128] inputs -> numpy f32, for a few head-chunk sizes, on
bf16-valued inputs (the lossless bf16 upload) and on the same inputs one ulp off
(the f32 upload)."""
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
exact_fn = ops.host_stage_bf16_exact
xb = [a.copy() for a in x[:2]]                  # bf16-valued q, k
xf = [a.copy() for a in x[:2]]
for a in xf:                                     # one ulp off: no longer bf16-exact, the f32 upload
    a.view(np.uint32)[...] |= 1
refs = {}
import os
MODES = os.environ.get("E2E_MODES", "f32-valued, no narrow attempt;f32-valued;bf16-valued").split(";")
for rep in range(2):
  for edge in [x == "1" for x in os.environ.get("E2E_EDGE", "1").split(",")]:
    ops._HOST_EDGE_CHUNKS = edge
    for mode in MODES:
        x[0][...], x[1][...] = (xb if mode == "bf16-valued" else xf)
        ops.host_stage_bf16_exact = (lambda d, s: False) if "no narrow" in mode else exact_fn
        for ch in [int(c) for c in os.environ.get("E2E_CHUNKS", "2,4").split(",")]:
            attention._HOST_CHUNK_HEADS = ch
            o = sla_attention(inp, cfg)
            key = mode.startswith("bf16")
            if key not in refs:
                refs[key] = o.copy()
            assert np.array_equal(o, refs[key]), "chunking / upload encoding changed the result"
            del o
            ts = []
            ops.HOST_PROFILE = {}
            for _ in range(4):
                t0 = time.perf_counter()
                o = sla_attention(inp, cfg)
                ts.append(time.perf_counter() - t0)
                del o
            m = ops.LAST_HOST_TRANSFER
            print(f"drop-in e2e {mode} edge={int(edge)} chunk {ch}: ms {[round(t * 1e3, 1) for t in ts]} median "
                  f"{np.median(ts) * 1e3:.1f}  h2d {m['h2d_bytes'] / 1e9:.2f} GB, narrow chunks "
                  f"{m['narrow_chunks']}/{m['chunks']}  host ms/call "
                  f"{ {k_: round(v_ * 250, 1) for k_, v_ in ops.HOST_PROFILE.items()} }", flush=True)
            ops.HOST_PROFILE = None
ops.host_stage_bf16_exact = exact_fn
