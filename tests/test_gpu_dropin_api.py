"""The drop-in modules (paper_2512_16093_b200.attention / .blockquant) against
the behaviours the reference's own suites pin (pkg/tests/test_attention.py,
test_blockquant.py; restated here, numpy in -> numpy out, on the GPU path):
exactness properties, known answers, tie rules, error texts and the pinned
fidelity thresholds."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def A():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2512_16093_b200 import _lib, attention
    _lib.load(require_device=True)
    return attention


@pytest.fixture(scope="module")
def B():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2512_16093_b200 import blockquant
    return blockquant


def gauss(A, seed, h, s, d):
    rng = np.random.default_rng(seed)
    return A.AttnInputs(*(rng.standard_normal((h, s, d), dtype=np.float32) for _ in range(3)))


def f64_attention(x):
    q, k, v = (t.astype(np.float64) for t in (x.q, x.k, x.v))
    lg = x.scale * q @ k.transpose(0, 2, 1)
    p = np.exp(lg - lg.max(-1, keepdims=True))
    return (p / p.sum(-1, keepdims=True)) @ v


# ------------------------------------------------------------ dense / smoothing

def test_reference_attention_properties(A):
    x = gauss(A, 0, 2, 1, 8)
    assert np.array_equal(A.reference_attention(x), x.v)                  # one key: output = v
    x = gauss(A, 3, 2, 128, 32)
    assert A.error_metrics(A.reference_attention(x), f64_attention(x).astype(np.float32))[1] <= 1e-6
    _, p = A.reference_attention(gauss(A, 5, 3, 64, 16), return_probs=True)
    assert np.abs(p.sum(-1) - 1).max() <= 1e-6
    rng = np.random.default_rng(1)
    k = np.repeat(rng.standard_normal((2, 1, 8)).astype(np.float32), 16, axis=1)
    q, v = (rng.standard_normal((2, 16, 8)).astype(np.float32) for _ in range(2))
    out = A.reference_attention(A.AttnInputs(q, k, v))                     # equal keys: column mean
    assert np.allclose(out, np.broadcast_to(v.mean(1, keepdims=True), out.shape), atol=1e-6)


def test_smooth_keys_properties(A):
    kc, km = A.smooth_keys(np.full((2, 16, 4), 3.25, np.float32))
    assert np.array_equal(kc, np.zeros((2, 16, 4), np.float32)) and np.allclose(km, 3.25)
    rng = np.random.default_rng(4)
    q = rng.standard_normal((2, 48, 16)).astype(np.float32)
    k = rng.standard_normal((2, 48, 16)).astype(np.float32) + 0.7
    kc, km = A.smooth_keys(k)
    rebuilt = q @ kc.transpose(0, 2, 1) + q @ km[:, :, None]
    assert A.error_metrics(rebuilt, q @ k.transpose(0, 2, 1))[1] <= 1e-5


# ----------------------------------------------------------- quantized attention

def test_quantized_attention_properties(A):
    x = gauss(A, 6, 4, 1, 16)
    assert np.array_equal(A.quantized_attention(x), x.v)
    rng = np.random.default_rng(7)
    k, v = (rng.standard_normal((2, 32, 8)).astype(np.float32) for _ in range(2))
    out = A.quantized_attention(A.AttnInputs(np.zeros((2, 32, 8), np.float32), k, v))
    assert np.allclose(out, np.broadcast_to(v.mean(1, keepdims=True), out.shape), atol=1e-6)


def test_quantized_attention_fidelity(A):
    worst_cos, worst_rel = 1.0, 0.0
    for seed in range(5, 15):
        x = gauss(A, seed, 4, 256, 64)
        cos, rel = A.error_metrics(A.quantized_attention(x), A.reference_attention(x))
        worst_cos, worst_rel = min(worst_cos, cos), max(worst_rel, rel)
    assert worst_cos >= 0.999 and worst_rel <= 5e-2
    x = gauss(A, 5, 4, 256, 64)
    assert A.error_metrics(A.quantized_attention(x, A.QuantAttnConfig(smooth_k=False)),
                           A.reference_attention(x))[0] >= 0.99


# -------------------------------------------------------------- pooling / top-k

def test_pool_block_means_known_answers(A):
    x = np.random.default_rng(8).standard_normal((2, 10, 4)).astype(np.float32)
    p = A.pool_block_means(x, 10)
    assert p.shape == (2, 1, 4) and np.allclose(p[:, 0], x.mean(1), atol=1e-6)
    x = np.random.default_rng(9).standard_normal((2, 7, 3)).astype(np.float32)
    assert np.array_equal(A.pool_block_means(x, 1), x)
    x = np.arange(5, dtype=np.float32).reshape(1, 5, 1)                   # blocks of 2, 2, 1
    assert np.array_equal(A.pool_block_means(x, 2), np.array([[[0.5], [2.5], [4.0]]], np.float32))


def test_select_topk_known_answers(A):
    rng = np.random.default_rng(10)
    m = A.select_topk_blocks(rng.standard_normal((2, 3, 4)).astype(np.float32),
                             rng.standard_normal((2, 5, 4)).astype(np.float32), A.SLAConfig(topk_ratio=1.0))
    assert np.array_equal(m.indices, np.broadcast_to(np.arange(5), (2, 3, 5)))
    scores = np.array([[[3, 1, 2, 0], [0, 0, 1, 5]]], np.float32)         # identity kp: scores = qp
    m = A.select_topk_blocks(scores, np.eye(4, dtype=np.float32)[None], A.SLAConfig(topk_ratio=0.5))
    assert m.indices[0].tolist() == [[0, 2], [2, 3]]
    m = A.select_topk_blocks(np.zeros((1, 1, 4), np.float32), np.ones((1, 8, 4), np.float32),
                             A.SLAConfig(topk_ratio=0.25))
    assert m.indices[0, 0].tolist() == [0, 1]                             # ties -> lower index


def test_select_topk_power_of_two_scale_invariance_and_complement(A):
    rng = np.random.default_rng(11)
    qp = rng.standard_normal((2, 6, 8)).astype(np.float32)
    kp = rng.standard_normal((2, 9, 8)).astype(np.float32)
    cfg = A.SLAConfig(topk_ratio=0.34)
    base = A.select_topk_blocks(qp, kp, cfg).indices
    for cq, ck in ((2.0, 1.0), (1.0, 0.25), (8.0, 4.0)):
        assert np.array_equal(A.select_topk_blocks(np.float32(cq) * qp, np.float32(ck) * kp, cfg).indices, base)
    m = A.select_topk_blocks(rng.standard_normal((2, 4, 8)).astype(np.float32),
                             rng.standard_normal((2, 10, 8)).astype(np.float32), A.SLAConfig(topk_ratio=0.3))
    c = m.complement()
    assert c.count == 10 - m.count
    both = np.sort(np.concatenate([m.indices, c.indices], -1), -1)
    assert np.array_equal(both, np.broadcast_to(np.arange(10), both.shape))


# --------------------------------------------------------------- linear branch

def test_linear_attention_properties(A):
    x = gauss(A, 13, 2, 32, 8)
    empty = A.BlockMask(16, 16, 2, np.empty((2, 2, 0), np.int64))
    num, den = A.linear_attention(x, empty)
    assert not num.any() and not den.any()
    x = gauss(A, 14, 3, 1, 8)
    num, den = A.linear_attention(x)
    assert np.allclose(num / den[..., None], x.v, atol=1e-6)
    x = gauss(A, 15, 2, 128, 16)
    _, den = A.linear_attention(x, A.BlockMask(32, 32, 4, np.full((2, 4, 1), 2, np.int64)))
    assert den.min() > 0


def test_linear_attention_masked_vs_f64(A):
    x = gauss(A, 16, 2, 40, 8)                                             # last kv block partial (16+16+8)
    mask = A.BlockMask(20, 16, 3, np.array([[[0, 2], [1, 2]], [[0, 1], [0, 2]]], np.int64))
    num, den = A.linear_attention(x, mask)
    phi = lambda t: np.where(t >= 0, t + 1.0, np.exp(np.minimum(t, 0.0)))
    for h in range(2):
        for n in range(2):
            rows = slice(20 * n, min(20 * n + 20, 40))
            pos = np.concatenate([np.arange(16 * b, min(16 * b + 16, 40)) for b in mask.indices[h, n]])
            pk, pq = phi(x.k[h, pos].astype(np.float64)), phi(x.q[h, rows].astype(np.float64))
            assert np.allclose(num[h, rows], pq @ (pk.T @ x.v[h, pos]), rtol=1e-5, atol=1e-5)
            assert np.allclose(den[h, rows], pq @ pk.sum(0), rtol=1e-5, atol=1e-5)


# ---------------------------------------------------------------- sla attention

@pytest.mark.parametrize("h,s,d,mix", [(2, 128, 16, 1.0), (1, 96, 8, 0.0), (3, 64, 32, 2.5), (2, 100, 16, 1.0),
                                       (2, 90, 8, 1.0)])
def test_sla_full_selection_equals_dense(A, h, s, d, mix):
    x = gauss(A, 20 + h + s, h, s, d)
    cfg = A.SLAConfig(q_block=32, kv_block=32, topk_ratio=1.0, linear_mix=mix, quantized_sparse_branch=False)
    assert A.error_metrics(A.sla_attention(x, cfg), A.reference_attention(x))[1] <= 1e-5


def test_sla_full_selection_ignores_mix_and_rejects_big_blocks(A):
    x = gauss(A, 21, 2, 64, 16)
    outs = [A.sla_attention(x, A.SLAConfig(32, 32, 1.0, m, False)) for m in (0.0, 1.0, 123.0)]
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[1], outs[2])
    with pytest.raises(ValueError):
        A.sla_attention(gauss(A, 22, 1, 16, 8), A.SLAConfig(q_block=64, kv_block=64))
    for bad in (dict(topk_ratio=0.0), dict(topk_ratio=1.5), dict(q_block=0), dict(linear_mix=-1.0)):
        with pytest.raises(ValueError):
            A.SLAConfig(**bad)


def test_sla_fidelity_gaussian_and_block_coherent(A):
    x = gauss(A, 9, 4, 512, 64)
    assert A.error_metrics(A.sla_attention(x, A.SLAConfig(topk_ratio=0.1)), A.reference_attention(x))[0] >= 0.58
    rng = np.random.default_rng(9)
    h, s, d, blk = 4, 512, 64, 64
    nb = s // blk
    centres = (3.0 * rng.standard_normal((h, nb, d))).astype(np.float32)
    k = np.repeat(centres, blk, axis=1) + 0.3 * rng.standard_normal((h, s, d)).astype(np.float32)
    tgt = np.repeat(rng.integers(0, nb, (h, nb)), blk, axis=1)
    q = centres[np.arange(h)[:, None], tgt] + 0.3 * rng.standard_normal((h, s, d)).astype(np.float32)
    v = rng.standard_normal((h, s, d)).astype(np.float32)
    x = A.AttnInputs(q, k, v)
    ref = A.reference_attention(x)
    assert A.error_metrics(A.sla_attention(x, A.SLAConfig(topk_ratio=0.1, quantized_sparse_branch=False)),
                           ref)[0] >= 0.9999
    assert A.error_metrics(A.sla_attention(x, A.SLAConfig(topk_ratio=0.1)), ref)[0] >= 0.99


# -------------------------------------------------------- flop report / metrics

def test_flop_report_and_instrumented_macs(A):
    assert A.attention_flop_report(4096, 64, 1).to_dict() == {"dense_flops": 4 * 4096 * 4096 * 64}
    r = A.attention_flop_report(4096, 64, 1, A.SLAConfig(topk_ratio=1.0))
    assert r.sparse_softmax_flops == r.dense_flops
    r = A.attention_flop_report(2560, 64, 1, A.SLAConfig(topk_ratio=0.1))
    assert r.sparse_softmax_flops * 10 == r.dense_flops and r.dense_to_sparse_ratio == 10.0
    cfg = A.SLAConfig(q_block=64, kv_block=64, topk_ratio=0.1)
    r = A.attention_flop_report(640, 32, 2, cfg)
    assert r.linear_branch_flops == 4 * 2 * 640 * 32 * 32
    assert r.selection_overhead_flops == 2 * 2 * 10 * 10 * 32 and r.sparse_softmax_flops <= r.dense_flops
    macs = A.instrumented_sparse_macs(gauss(A, 24, 2, 640, 32), cfg)
    assert macs["total_macs"] * 10 == macs["dense_macs"] and 2 * macs["total_macs"] == r.sparse_softmax_flops


def test_error_metrics_semantics(A):
    a = np.random.default_rng(0).standard_normal((3, 4)).astype(np.float32)
    assert A.error_metrics(a, a) == (1.0, 0.0)
    a = np.random.default_rng(1).standard_normal(16).astype(np.float32)
    cos, rel = A.error_metrics(-a, a)
    assert abs(cos + 1) < 1e-7 and abs(rel - 2) < 1e-7
    b = np.zeros(4, np.float32)
    b[0] = 1.0
    a = b.copy()
    a[1] = 0.1
    assert abs(A.error_metrics(a, b)[1] - 0.1) < 1e-7
    for x, y in ((np.zeros(4, np.float32), np.ones(4, np.float32)), (np.ones(4, np.float32), np.zeros(4, np.float32))):
        with pytest.raises(ValueError):
            A.error_metrics(x, y)


# ------------------------------------------------------------------ blockquant

def _dequant_loop(bq):
    out = np.empty((bq.rows, bq.cols), np.float32)
    b = bq.block
    for i in range(bq.scales.shape[0]):
        for j in range(bq.scales.shape[1]):
            out[i * b:(i + 1) * b, j * b:(j + 1) * b] = np.asarray(bq.q)[i * b:(i + 1) * b, j * b:(j + 1) * b] \
                .astype(np.float32) * np.asarray(bq.scales)[i, j]
    return out


def test_blockquant_known_answers(B):
    z = B.quantize_blockwise(np.zeros((128, 128), np.float32))
    assert not np.asarray(z.q).any() and not np.asarray(z.scales).any()
    assert not np.asarray(B.dequantize_blockwise(z)).any()
    c = np.float32(0.731)
    m = np.full((128, 128), 127 * c, np.float32)
    bq = B.quantize_blockwise(m)                                          # constant block: a fixed point
    assert (np.asarray(bq.q) == 127).all() and np.asarray(bq.scales).shape == (1, 1)
    assert np.allclose(np.asarray(bq.scales)[0, 0], c, rtol=1e-6)
    assert np.array_equal(np.asarray(B.dequantize_blockwise(bq)), m)
    s = np.float32(0.01)
    ext = B.BlockQuantized(rows=2, cols=2, block=128, q=np.array([[127, -127], [127, -127]], np.int8),
                           scales=np.array([[s]], np.float32))
    assert np.array_equal(np.asarray(B.dequantize_blockwise(ext)), np.array([[127 * s, -127 * s]] * 2, np.float32))


def test_blockquant_roundtrip_bound_and_brute_force_dequant(B):
    m = np.random.default_rng(7).standard_normal((256, 256), dtype=np.float32)
    bq = B.quantize_blockwise(m)
    err = np.abs(m - np.asarray(B.dequantize_blockwise(bq)))
    assert (err <= B._expand_scales(np.asarray(bq.scales), 128, 256, 256) / 2 + np.spacing(np.abs(m))).all()
    m = np.random.default_rng(8).standard_normal((300, 200), dtype=np.float32)     # edge blocks
    bq = B.quantize_blockwise(m)
    assert np.array_equal(np.asarray(B.dequantize_blockwise(bq)), _dequant_loop(bq))


@pytest.mark.parametrize("seed", [0, 17, 4242, 9999])
def test_blockquant_requantize_idempotent(B, seed):
    rng = np.random.default_rng(seed)
    m = (rng.standard_normal((64, 96)) * rng.uniform(1e-3, 1e3)).astype(np.float32)
    cfg = B.BlockQuantConfig(block=32)
    first = B.quantize_blockwise(m, cfg)
    again = B.quantize_blockwise(np.asarray(B.dequantize_blockwise(first)), cfg)
    assert np.array_equal(np.asarray(first.q), np.asarray(again.q))
    assert np.array_equal(np.asarray(first.scales), np.asarray(again.scales))


@pytest.mark.parametrize("c", [2.0, 0.5, 8.0, 0.0625])
def test_blockquant_power_of_two_scaling(B, c):
    m = np.random.default_rng(9).standard_normal((130, 70), dtype=np.float32)
    base, scaled = B.quantize_blockwise(m), B.quantize_blockwise(np.float32(c) * m)
    assert np.array_equal(np.asarray(scaled.q), np.asarray(base.q))
    assert np.array_equal(np.asarray(scaled.scales), np.float32(c) * np.asarray(base.scales))


def test_blockquant_rejects_non_finite_and_mismatches(B):
    m = np.zeros((4, 4), np.float32)
    m[1, 2] = np.inf
    with pytest.raises(ValueError):
        B.quantize_blockwise(m)
    rng = np.random.default_rng(4)
    a = B.quantize_blockwise(rng.standard_normal((8, 16), dtype=np.float32))
    with pytest.raises(ValueError, match="inner dims"):
        B.w8a8_matmul(a, B.quantize_blockwise(rng.standard_normal((8, 8), dtype=np.float32)))
    with pytest.raises(ValueError, match="block"):
        B.w8a8_matmul(a, B.quantize_blockwise(rng.standard_normal((16, 8), dtype=np.float32),
                                              B.BlockQuantConfig(block=64)))
    w = B.quantize_blockwise(rng.standard_normal((32, 16), dtype=np.float32))
    with pytest.raises(ValueError):
        B.quantized_linear_forward(np.zeros((4, 8), np.float32), w)


def test_w8a8_known_answers(B):
    rng = np.random.default_rng(1)
    a = B.quantize_blockwise(rng.standard_normal((64, 64), dtype=np.float32))
    assert not np.asarray(B.w8a8_matmul(a, B.quantize_blockwise(np.zeros((64, 32), np.float32)))).any()
    a = B.quantize_blockwise(np.eye(128, dtype=np.float32))
    b = B.quantize_blockwise(np.random.default_rng(2).standard_normal((128, 128), dtype=np.float32))
    want = np.asarray(B.dequantize_blockwise(a)) @ np.asarray(B.dequantize_blockwise(b))
    assert np.allclose(np.asarray(B.w8a8_matmul(a, b)), want, atol=1e-6)
    rng = np.random.default_rng(11)
    a, b = (B.quantize_blockwise(rng.standard_normal((256, 256), dtype=np.float32)) for _ in range(2))
    assert np.abs(np.asarray(B.w8a8_matmul(a, b)) - _dequant_loop(a) @ _dequant_loop(b)).max() <= 1e-3


def test_w8a8_equals_int64_segment_order(B):
    rng = np.random.default_rng(3)
    cfg = B.BlockQuantConfig(block=64)
    a = B.quantize_blockwise(rng.standard_normal((96, 192), dtype=np.float32), cfg)
    b = B.quantize_blockwise(rng.standard_normal((192, 80), dtype=np.float32), cfg)
    aq, bqq, sa, sb = (np.asarray(t) for t in (a.q, b.q, a.scales, b.scales))
    out = np.zeros((96, 80), np.float32)
    for kb in range(sa.shape[1]):
        lo, hi = 64 * kb, min(64 * kb + 64, 192)
        seg = (aq[:, lo:hi].astype(np.int64) @ bqq[lo:hi].astype(np.int64)).astype(np.float32)
        seg *= np.repeat(sa[:, kb], [64, 32])[:, None]
        seg *= np.repeat(sb[kb], [64, 16])[None, :]
        out += seg
    assert np.array_equal(np.asarray(B.w8a8_matmul(a, b)), out)


def test_quantized_linear_forward_semantics(B):
    rng = np.random.default_rng(5)
    w = B.quantize_blockwise(rng.standard_normal((32, 16), dtype=np.float32))
    bias = rng.standard_normal(16, dtype=np.float32)
    assert np.array_equal(np.asarray(B.quantized_linear_forward(np.zeros((4, 32), np.float32), w, bias)),
                          np.tile(bias, (4, 1)))
    rng = np.random.default_rng(6)
    x = rng.standard_normal((8, 32), dtype=np.float32)
    w = B.quantize_blockwise(rng.standard_normal((32, 16), dtype=np.float32))
    assert np.array_equal(np.asarray(B.quantized_linear_forward(x, w)),
                          np.asarray(B.w8a8_matmul(B.quantize_blockwise(x), w)))
    rng = np.random.default_rng(13)
    x = rng.standard_normal((128, 128), dtype=np.float32)
    wf = rng.standard_normal((128, 128), dtype=np.float32)
    got = np.asarray(B.quantized_linear_forward(x, B.quantize_blockwise(wf)))
    assert np.linalg.norm(got - x @ wf) / np.linalg.norm(x @ wf) <= 0.02


def test_compression_ratio_accounting(B):
    bq = B.quantize_blockwise(np.random.default_rng(0).standard_normal((128, 128)).astype(np.float32))
    assert B.compression_ratio(bq, 2.0) == (128 * 128 + 4) / (2 * 128 * 128)
    assert abs(B.compression_ratio(bq, 4.0) - 0.25006) < 1e-4
    assert B.compression_ratio(B.quantize_blockwise(np.ones((1, 1), np.float32)), 1.0) == 5.0
    with pytest.raises(ValueError):
        B.compression_ratio(bq, 0.0)


# --------------------------------------------------------------------- sampler

@pytest.fixture(scope="module")
def S():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2512_16093_b200 import sampler
    return sampler


def test_norms_known_answers_and_f64(S, A):
    assert np.array_equal(np.asarray(S.rmsnorm(np.zeros((3, 8), np.float32), np.ones(8, np.float32))),
                          np.zeros((3, 8), np.float32))
    x = np.ones((1, 16), np.float32)
    assert np.abs(np.asarray(S.rmsnorm(x, np.ones(16, np.float32), eps=1e-12)) - x).max() <= 1e-6
    rng = np.random.default_rng(0)
    x, g = rng.standard_normal((64, 32)).astype(np.float32), rng.standard_normal(32).astype(np.float32)
    x64 = x.astype(np.float64)
    want = (x64 / np.sqrt((x64 ** 2).mean(-1, keepdims=True) + 1e-6) * g).astype(np.float32)
    assert A.error_metrics(np.asarray(S.rmsnorm(x, g)), want)[1] <= 1e-6
    gain, off = (np.random.default_rng(i).standard_normal(8).astype(np.float32) for i in (1, 2))
    assert np.array_equal(np.asarray(S.layernorm(np.full((4, 8), 2.5, np.float32), gain, off)), np.tile(off, (4, 1)))
    x = np.random.default_rng(3).standard_normal((32, 64)).astype(np.float32) * 5 + 3
    out = np.asarray(S.layernorm(x, np.ones(64, np.float32), np.zeros(64, np.float32)))
    assert np.abs(out.mean(-1)).max() <= 1e-5 and np.abs(out.var(-1) - 1).max() <= 1e-4
    rng = np.random.default_rng(4)
    x, g, o = (rng.standard_normal(sh).astype(np.float32) for sh in ((64, 32), 32, 32))
    x64 = x.astype(np.float64)
    mu = x64.mean(-1, keepdims=True)
    want = ((x64 - mu) / np.sqrt(((x64 - mu) ** 2).mean(-1, keepdims=True) + 1e-6) * g + o).astype(np.float32)
    assert A.error_metrics(np.asarray(S.layernorm(x, g, o)), want)[1] <= 1e-6
    for fn, args in ((S.rmsnorm, ()), (S.layernorm, (np.zeros(4, np.float32),))):
        with pytest.raises(ValueError):
            fn(np.ones((2, 4), np.float32), np.ones(4, np.float32), *args, eps=0.0)


def _gauss_weights(S, seed, d, mult=4):
    rng = np.random.default_rng(seed)
    mat = lambda r, c: rng.standard_normal((r, c), dtype=np.float32) / np.float32(np.sqrt(r))
    return S.ToyBlockWeights(rms_gain=rng.standard_normal(d, dtype=np.float32) * 0.1 + 1,
                             ln_gain=rng.standard_normal(d, dtype=np.float32) * 0.1 + 1,
                             ln_offset=rng.standard_normal(d, dtype=np.float32) * 0.1,
                             qkv=mat(d, 3 * d), out_proj=mat(d, d), mlp_in=mat(d, mult * d),
                             mlp_out=mat(mult * d, d), sigma_emb=rng.standard_normal(d, dtype=np.float32) * 0.01)


def test_toy_block_semantics(S, A):
    d = 32
    zero = S.ToyBlockWeights(**{n: np.zeros(sh, np.float32) for n, sh in (
        ("rms_gain", d), ("ln_gain", d), ("ln_offset", d), ("qkv", (d, 3 * d)), ("out_proj", (d, d)),
        ("mlp_in", (d, 4 * d)), ("mlp_out", (4 * d, d)), ("sigma_emb", d))})
    x = np.random.default_rng(5).standard_normal((16, d)).astype(np.float32)
    assert np.array_equal(np.asarray(S.toy_block_forward(x, 7.0, zero, heads=4)), x)      # zero weights: identity
    with pytest.raises(ValueError):
        S.toy_block_forward(np.zeros((4, 30), np.float32), 1.0, S.ToyBlockWeights(
            **{n: np.zeros(sh, np.float32) for n, sh in (("rms_gain", 30), ("ln_gain", 30), ("ln_offset", 30),
               ("qkv", (30, 90)), ("out_proj", (30, 30)), ("mlp_in", (30, 120)), ("mlp_out", (120, 30)),
               ("sigma_emb", 30))}), heads=4)
    w = _gauss_weights(S, 6, 128)
    x = np.random.default_rng(7).standard_normal((256, 128)).astype(np.float32)
    dense = np.asarray(S.toy_block_forward(x, 1.5, w, heads=4, attn_mode="dense"))
    sla = np.asarray(S.toy_block_forward(x, 1.5, w, heads=4, attn_mode="sla",
                                         sla_cfg=A.SLAConfig(64, 64, 1.0, 1.0, False)))
    assert A.error_metrics(sla, dense)[1] <= 1e-5
    from paper_2512_16093_b200.blockquant import quantize_blockwise
    w = _gauss_weights(S, 13, 128)
    wq = S.ToyBlockWeights(rms_gain=w.rms_gain, ln_gain=w.ln_gain, ln_offset=w.ln_offset,
                           qkv=quantize_blockwise(w.qkv), out_proj=quantize_blockwise(w.out_proj),
                           mlp_in=quantize_blockwise(w.mlp_in), mlp_out=quantize_blockwise(w.mlp_out),
                           sigma_emb=w.sigma_emb)
    x = np.random.default_rng(13).standard_normal((256, 128)).astype(np.float32)
    dense = np.asarray(S.toy_block_forward(x, 2.0, w, heads=4, attn_mode="dense"))
    quant = np.asarray(S.toy_block_forward(x, 2.0, wq, heads=4, attn_mode="quantized"))
    assert A.error_metrics(quant, dense)[0] >= 0.97


def test_schedule_semantics(S):
    s1 = S.make_schedule(1, sigma_max=80.0, sigma_min=0.5)
    assert np.array_equal(s1.sigmas, np.array([80.0, 0.0], np.float32)) and s1.num_steps == 1
    s = S.make_schedule(3, sigma_max=80.0, sigma_min=0.5).sigmas.astype(np.float64)
    assert s[0] == 80.0 and abs(s[2] - 0.5) < 1e-6 and s[3] == 0.0
    assert abs(s[1] / s[0] - s[2] / s[1]) < 1e-6 and abs(s[1] - np.sqrt(40.0)) < 1e-4
    for n, smax, smin in ((100, 80.0, 0.5), (7, 500.0, 1e-3), (200, 1.0, 0.9)):
        sc = S.make_schedule(n, smax, smin)
        assert sc.num_steps == n and (np.diff(sc.sigmas) < 0).all() and sc.sigmas[-1] == 0.0
    for bad in (lambda: S.make_schedule(3, sigma_max=0.5, sigma_min=0.5), lambda: S.make_schedule(0),
                lambda: S.Schedule(np.array([1.0, 2.0, 0.0], np.float32))):
        with pytest.raises(ValueError):
            bad()


def test_consistency_sample_semantics(S):
    c = np.float32(3.75)
    for n in (1, 2, 5):
        out = S.consistency_sample(lambda x, s: np.full_like(x, c), S.make_schedule(n), (4, 4), seed=0)
        assert np.array_equal(out, np.full((4, 4), c, np.float32))
    for n in (1, 3, 4, 100):
        calls = []
        S.consistency_sample(lambda x, s: (calls.append(s), x * np.float32(0.9))[1], S.make_schedule(n), (2, 2), 5)
        assert len(calls) == n
    seen = {}

    def first(x, s):
        seen.setdefault("x", np.array(x, copy=True))
        seen.setdefault("s", s)
        return np.zeros_like(x)
    S.consistency_sample(first, S.make_schedule(1, sigma_max=10.0, sigma_min=1.0), (8,), seed=3)
    assert seen["s"] == 10.0 and np.array_equal(seen["x"], np.float32(10.0) * S.step_noise(3, 0, (8,)))
    a = (np.random.default_rng(8).standard_normal((6, 6)) * 0.3).astype(np.float32)
    lin = lambda x, s: (a @ x.T).T.astype(np.float32)
    sc = S.make_schedule(3, sigma_max=4.0, sigma_min=0.25)
    x = np.float32(sc.sigmas[0]) * S.step_noise(11, 0, (2, 6))
    for i in (1, 2):
        x = lin(x, None) + np.float32(sc.sigmas[i]) * S.step_noise(11, i, (2, 6))
    assert np.allclose(S.consistency_sample(lin, sc, (2, 6), 11), lin(x, None), atol=1e-6)
    tanh = lambda x, s: np.tanh(x)
    assert np.array_equal(S.consistency_sample(tanh, S.make_schedule(4), (16, 8), 9),
                          S.consistency_sample(tanh, S.make_schedule(4), (16, 8), 9))
    with pytest.raises(ValueError):
        S.consistency_sample(lambda x, s: np.zeros((1,), np.float32), S.make_schedule(2), (4,), seed=0)


def test_two_expert_semantics(S):
    sc = S.make_schedule(3, 80.0, 0.5)
    hi_, lo_ = (lambda x, s: np.full_like(x, np.float32(2.0))), (lambda x, s: np.full_like(x, np.float32(-1.0)))
    mid = float(np.sqrt(sc.sigmas[1] * sc.sigmas[2]))
    for boundary, want_sw, want in ((1000.0, 0, -1.0), (0.01, 0, 2.0), (mid, 1, -1.0)):
        out, sw = S.two_expert_sample(S.TwoExpertConfig(boundary, hi_, lo_), sc, (4,), seed=0)
        assert sw == want_sw and np.array_equal(out, np.full((4,), want, np.float32))
    with pytest.raises(ValueError):
        S.TwoExpertConfig(0.0, hi_, lo_)


def test_quantized_weights_take_the_w8a8_path(S, A):
    layers = S.make_random_weights(64, num_layers=1, seed=4)
    x = np.random.default_rng(1).standard_normal((16, 64)).astype(np.float32)
    dense = np.asarray(S.ToyModel(layers=layers, heads=2)(x, 0.5))
    quant = np.asarray(S.ToyModel(layers=S.quantize_weights(layers), heads=2)(x, 0.5))
    assert A.error_metrics(quant, dense)[0] >= 0.97 and not np.array_equal(quant, dense)
