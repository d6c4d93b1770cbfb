"""GPU parity at the headline shapes.

The fused attention OUTPUT is checked where the bench times it:
* cfg4 (BASELINE configs[3]: 75600 tokens, nkv 1182 with a ragged last kv
  block of 16 tokens, a ragged last q-block of 80 rows, 119 selected blocks
  per row) on two full-length heads against the CPU oracle, Gaussian and
  block-coherent (sparse-dominated) inputs, linear_mix 1 and 0, through the
  device op the bench times (bf16 in / bf16 out) and through the drop-in
  ``attention.sla_attention`` (numpy f32 in / f32 out);
* one head of cfg4 and of cfg3 (q_block 128 and the reference default 64)
  against row subsamples of the REFERENCE's own output
  (tests/golden/headline.npz, written by make_golden.py from turbobench);
* the four cfg2 W8A8 shapes (BASELINE configs[1]) bit-exact in exact mode on
  the first, a middle and the ragged last row block.

Tolerances (north star): cos >= 0.999 and rel-L1 <= 1e-2 for attention
outputs; bit-exact (array_equal) for the W8A8 exact mode.
"""
import numpy as np
import pytest
import torch

import gen
from conftest import load_golden
from oracle import oracle as O

pytestmark = pytest.mark.gpu

COS_MIN, REL_L1_MAX = 0.999, 1e-2
L4, L3, D = 75600, 32760, 128


@pytest.fixture(scope="module")
def tb():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2512_16093_b200 import _lib, ops
    _lib.load(require_device=True)
    return ops


def dev(a, bf16=False):
    t = torch.from_numpy(np.ascontiguousarray(a, np.float32)).cuda()
    return t.to(torch.bfloat16) if bf16 else t


def check(got, want, what):
    cos, _, rel1 = O.error_metrics(np.asarray(got, np.float32), np.asarray(want, np.float32))
    assert cos >= COS_MIN and rel1 <= REL_L1_MAX, (what, cos, rel1)
    return cos, rel1


@pytest.fixture(scope="module")
def cfg4_inputs():
    return {"G": gen.gaussian_qkv(2, 2, L4, D, bf16=True),
            "B": gen.block_coherent_qkv(13, 2, L4, D, blk=64, bf16=True)}


@pytest.mark.parametrize("g", ["G", "B"])
@pytest.mark.parametrize("mix", [1.0, 0.0])
def test_cfg4_two_heads_vs_oracle(tb, cfg4_inputs, g, mix):
    """The bench's exact device path (bf16 in, bf16 out, q_block 128 / kv 64)
    and the drop-in (numpy f32 in, f32 out) on two full cfg4 heads."""
    from paper_2512_16093_b200.attention import AttnInputs, SLAConfig, sla_attention
    q, k, v = cfg4_inputs[g]
    want = O.sla_attention(q, k, v, 128, 64, 0.1, mix)
    got = tb.sla_attention(dev(q, True), dev(k, True), dev(v, True), 128, 64, 0.1, mix,
                           out_dtype=torch.bfloat16)
    check(got.float().cpu().numpy(), want, ("ops bf16", g, mix))
    # the ragged tail on its own: last q-block (80 rows) sees the 16-token kv block
    check(got.float().cpu().numpy()[:, -80:], want[:, -80:], ("ragged tail", g, mix))
    got2 = sla_attention(AttnInputs(q, k, v), SLAConfig(q_block=128, kv_block=64, topk_ratio=0.1, linear_mix=mix))
    assert got2.dtype == np.float32 and got2.shape == q.shape
    check(got2, want, ("drop-in f32", g, mix))


@pytest.mark.parametrize("case", gen.HEADLINE_CASES, ids=lambda c: c[0])
def test_headline_vs_reference_golden(tb, case):
    """Row subsamples of turbobench's own sla_attention output (one full-length
    head) against the drop-in and the bf16 device op."""
    from paper_2512_16093_b200.attention import AttnInputs, SLAConfig, sla_attention
    name, g_, seed, h, s, d, qb, kvb, ratio, mixes = case
    gold = load_golden("headline")
    rows = gold[name + ".rows_idx"]
    q, k, v = gen.make_inputs(g_, seed, h, s, d)
    for mix in mixes:
        want = gold[f"{name}.mix{mix:g}.rows"]
        got = sla_attention(AttnInputs(q, k, v), SLAConfig(q_block=qb, kv_block=kvb, topk_ratio=ratio,
                                                           linear_mix=mix))
        check(got[:, rows], want, (name, mix, "drop-in"))
        got_b = tb.sla_attention(dev(q, True), dev(k, True), dev(v, True), qb, kvb, ratio, mix,
                                 out_dtype=torch.bfloat16)
        check(got_b.float().cpu().numpy()[:, rows], want, (name, mix, "ops bf16"))


def test_cfg3_one_head_vs_oracle_both_q_blocks(tb):
    """cfg3 (BASELINE configs[2], Wan2.1-1.3B layer: 32760 tokens, last kv
    block 56 tokens) at q_block 128 and the reference default 64."""
    q, k, v = gen.gaussian_qkv(1, 1, L3, D, bf16=True)
    for qb in (128, 64):
        for mix in (1.0, 0.0):
            want = O.sla_attention(q, k, v, qb, 64, 0.1, mix)
            got = tb.sla_attention(dev(q, True), dev(k, True), dev(v, True), qb, 64, 0.1, mix)
            check(got.cpu().numpy(), want, (qb, mix))


CFG2 = [(1536, 1536), (1536, 4608), (1536, 8960), (8960, 1536)]


@pytest.mark.parametrize("K,N", CFG2, ids=lambda x: str(x))
def test_w8a8_cfg2_all_shapes_bit_exact(tb, K, N):
    """BASELINE configs[1] (M = 32760 tokens) in exact mode: rows of the first,
    a middle and the ragged last (120-row) block bit-exact against the
    oracle's reference-order restatement (blockquant.py:132-161), including
    K = 8960 (70 k-blocks); fast mode within 1e-4 rel-L1 of it."""
    M = 32760
    x = gen.gaussian_matrix(60 + K % 7, M, K, bf16=True)
    w = gen.gaussian_matrix(61 + N % 5, K, N, 1.0 / np.sqrt(K))
    wq, ws = O.quantize_blockwise(w, 128)
    bt = tb.transpose_codes(torch.from_numpy(wq).cuda())
    xq, xs = tb.quantize_blockwise(dev(x, bf16=True), 128)
    got = tb.w8a8_gemm(xq, xs, bt, dev(ws), 128).cpu().numpy()
    fast = tb.w8a8_gemm(xq, xs, bt, dev(ws), 128, exact=False).cpu().numpy()
    xq_n, xs_n = xq.cpu().numpy(), xs.cpu().numpy()
    for rb in (0, 131, 255):
        r0, r1 = rb * 128, min(rb * 128 + 128, M)
        want = O.w8a8(xq_n[r0:r1], xs_n[rb:rb + 1], wq, ws, 128)
        assert np.array_equal(got[r0:r1], want), (K, N, rb, int((got[r0:r1] != want).sum()))
        cos, _, rel1 = O.error_metrics(fast[r0:r1], want)
        assert cos >= 0.99999 and rel1 <= 1e-4, (K, N, rb, cos, rel1)


@pytest.mark.parametrize("block", [1100, 2048])
def test_w8a8_large_block_matches_int64_order(tb, block):
    """Block edges above the reference's f32-exact bound (1040) take its int64
    path (blockquant.py:119-129): exact int segment, one f32 rounding."""
    M, K, N = 300, 2 * block + 37, 260
    x = gen.gaussian_matrix(70, M, K)
    w = gen.gaussian_matrix(71, K, N, 1.0 / np.sqrt(K))
    wq, ws = O.quantize_blockwise(w, block)
    xq, xs = O.quantize_blockwise(x, block)
    want = O.w8a8(xq, xs, wq, ws, block)
    bt = tb.transpose_codes(torch.from_numpy(wq).cuda())
    got = tb.w8a8_gemm(torch.from_numpy(xq).cuda(), dev(xs), bt, dev(ws), block).cpu().numpy()
    assert np.array_equal(got, want), int((got != want).sum())


def test_w8a8_temporary_operands_survive_until_launch(tb):
    """Non-contiguous scales and a strided bf16 bias: each argument is converted
    to a fresh temporary inside the argument list, and every temporary must
    stay alive until the kernel is enqueued (ops.ptr keeps it) -- otherwise
    the caching allocator may hand one temporary's block to the next and the
    kernel reads overwritten scales."""
    M, K, N = 512, 256, 512
    x = gen.gaussian_matrix(80, M, K)
    w = gen.gaussian_matrix(81, K, N, 1.0 / np.sqrt(K))
    bias = gen.round_bf16(gen.gaussian_matrix(82, 1, N)[0])
    wq, ws = O.quantize_blockwise(w, 128)
    xq, xs = O.quantize_blockwise(x, 128)
    want = (O.w8a8(xq, xs, wq, ws, 128) + bias[None, :]).astype(np.float32)
    bt = tb.transpose_codes(torch.from_numpy(wq).cuda())
    aq = torch.from_numpy(xq).cuda()
    for _ in range(3):
        xs_nc = dev(xs.T.copy()).t()                               # non-contiguous views
        ws_nc = dev(ws.T.copy()).t()
        b_nc = dev(np.stack([bias, bias], 1), bf16=True).t()[0]     # strided bf16
        assert not (xs_nc.is_contiguous() or ws_nc.is_contiguous() or b_nc.is_contiguous())
        got = tb.w8a8_gemm(aq, xs_nc, bt, ws_nc, 128, bias=b_nc).cpu().numpy()
        assert np.array_equal(got, want), int((got != want).sum())
