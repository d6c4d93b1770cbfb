"""kv_part (with the K pool) alone at cfg4 under CUDA-graph replay; tools only."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_16093_b200 import ops  # noqa: E402

H, L, D = 40, 75600, 128
g = torch.Generator(device="cuda").manual_seed(0)
k, v = (torch.randn((H, L, D), generator=g, device="cuda").to(torch.bfloat16) for _ in range(2))
fn = lambda: ops.linear_kv_part(k, v, 64, pool=True)  # noqa: E731
for _ in range(3):
    fn()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    fn()
e1.record()
torch.cuda.synchronize()
print(f"{os.environ.get('TB200_LIB', 'libtb200.so').split('/')[-1]} per_sm={os.environ.get('TB_KVP_PER_SM', '-')}: "
      f"{e0.elapsed_time(e1) / 20:.3f} ms")
