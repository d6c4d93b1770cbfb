"""cfg5 norm-fed quantization (tools only): fused tb_add_norm_quant vs
tb_add_norm + quantize_blockwise at [75600, 5120] f32, RMSNorm and LayerNorm,
CUDA events, median of 10."""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_16093_b200 import ops  # noqa: E402

R, C = 75600, 5120
g = torch.Generator(device="cuda").manual_seed(0)
x, y = (torch.randn((R, C), generator=g, device="cuda") for _ in range(2))
emb = torch.randn(C, generator=g, device="cuda")
gain, off = torch.rand(C, generator=g, device="cuda") + 0.5, torch.randn(C, generator=g, device="cuda") * 0.1


def t(fn, n=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(n):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


for ln in (False, True):
    kw = dict(layer_norm=True, gain=gain, offset=off) if ln else dict(gain=gain)
    e = None if ln else emb
    a = t(lambda: ops.add_norm_quant(x, y, e, 0.5, **kw))
    b = t(lambda: ops.quantize_blockwise(ops.add_norm(x, y, e, 0.5, **kw)[1], 128, check_finite=False))
    print(f"{'LayerNorm' if ln else 'RMSNorm'}: fused add_norm_quant {a:.3f} ms, add_norm + quantize {b:.3f} ms "
          f"(fused {13 * R * C / a / 1e6:.0f} GB/s of 13 B/elt)")
