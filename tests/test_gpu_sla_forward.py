"""The single-call C-ABI pipeline (tb_sla_forward) against the
Python-orchestrated device op and the CPU oracle.

tb_sla_forward issues the same kernels as ops.sla_attention from one C entry
point (helper streams forked / joined with events, intermediates in one
workspace), so its output must equal ops.sla_attention bit for bit; the
oracle comparison uses the north-star tolerance (cos >= 0.999, rel-L1 <= 1e-2).
"""
import numpy as np
import pytest
import torch

import gen
from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tb():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2512_16093_b200 import _lib, ops
    _lib.load(require_device=True)
    return ops


@pytest.mark.parametrize("L", [5000, 200])
@pytest.mark.parametrize("qb", [128, 64])
@pytest.mark.parametrize("bf16", [True, False])
@pytest.mark.parametrize("mix", [1.0, 0.0])
def test_sla_forward_equals_device_op(tb, qb, bf16, mix, L):
    # 5000: ragged last kv block (5000 % 64 = 8); 200: two q-blocks, four kv blocks, one selected
    q, k, v = gen.gaussian_qkv(21, 3, L, 128, bf16=True)
    dt = torch.bfloat16 if bf16 else torch.float32
    dq, dk, dv = (torch.from_numpy(t).cuda().to(dt) for t in (q, k, v))
    want = tb.sla_attention(dq, dk, dv, qb, 64, 0.1, mix, out_dtype=torch.float32)
    got = tb.sla_forward(dq, dk, dv, qb, 64, 0.1, mix, out_dtype=torch.float32)
    torch.cuda.synchronize()
    assert torch.equal(got, want)
    ref = O.sla_attention(q, k, v, qb, 64, 0.1, mix)
    cos, _, rel1 = O.error_metrics(got.cpu().numpy(), ref)
    assert cos >= 0.999 and rel1 <= 1e-2, (cos, rel1)


def test_sla_forward_graph_capture_and_bf16_out(tb):
    """Helper streams fork / join by events: the call captures into a CUDA graph."""
    q, k, v = gen.gaussian_qkv(22, 2, 4096, 128, bf16=True)
    dq, dk, dv = (torch.from_numpy(t).cuda().to(torch.bfloat16) for t in (q, k, v))
    want = tb.sla_attention(dq, dk, dv, 128, 64, 0.1, 1.0, out_dtype=torch.bfloat16)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        tb.sla_forward(dq, dk, dv, 128, 64, 0.1, 1.0, out_dtype=torch.bfloat16)   # warm-up (allocator, attributes)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        out = tb.sla_forward(dq, dk, dv, 128, 64, 0.1, 1.0, out_dtype=torch.bfloat16)
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(out, want)


def test_sla_forward_rejects_outside_envelope(tb):
    q = torch.zeros((1, 512, 64), device="cuda", dtype=torch.bfloat16)
    with pytest.raises(RuntimeError, match="envelope"):
        tb.sla_forward(q, q, q, 64, 64, 0.1, 1.0)
    q = torch.zeros((1, 512, 128), device="cuda", dtype=torch.bfloat16)
    with pytest.raises(ValueError):
        tb.sla_forward(q, q, q, 64, 64, 0.0, 1.0)
