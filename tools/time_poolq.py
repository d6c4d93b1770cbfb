"""Time the cfg4 pool+quant passes (Q: block 128 with pooling; K codes: block 64 centred; K pool)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_16093_b200 import ops  # noqa: E402

H, L, D = 40, 75600, 128
g = torch.Generator(device="cuda").manual_seed(0)
q, k = (torch.randn((H, L, D), generator=g, device="cuda").to(torch.bfloat16) for _ in range(2))
km = ops.kmean(k)
cases = {"Q pass": lambda: ops.pool_quant_tokens(q, 128, None, pool=True),
         "K codes": lambda: ops.pool_quant_tokens(k, 64, km, pool=False),
         "K pool": lambda: ops.pool_tokens_t(k, 64)}
for name, fn in cases.items():
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        fn()
    e1.record()
    torch.cuda.synchronize()
    print(f"{os.environ.get('TB200_LIB', 'libtb200.so').split('/')[-1]} {name}: {e0.elapsed_time(e1) / 20:.3f} ms")
