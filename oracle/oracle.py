"""CPU oracle for the TurboDiffusion hot path -- TEST INFRASTRUCTURE ONLY.

This module restates the reference algorithm (/root/reference/pkg/src/
turbobench, pure numpy) so that parity tests, ``__graft_entry__.smoke()`` and
``bench.py``'s cpu_baseline / ``--impl reference`` legs can check and time the
GPU product against it on a box where /root/reference does not exist.
Nothing in ``paper_2512_16093_b200`` imports it; the product fails loudly if
its CUDA library is missing instead of falling back here.

Split:
* order-sensitive integer/byte/index work (block pooling, k_mean, INT8
  codes and scales, block scores + top-k, W8A8 segments) runs through
  ``liboracle.so`` (oracle/tb_oracle.c), whose summation orders are pinned
  against golden vectors produced by the reference itself
  (tests/golden/make_golden.py, tests/test_oracle_golden.py);
* floating-point branches (sparse softmax, linear attention, combine,
  norms, sampler) are numpy restatements, checked against the same goldens
  within tolerance.

Parity status: pinned (tests/test_oracle_golden.py, golden vectors from the
reference run in the build container).
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

_f32p = np.ctypeslib.ndpointer(dtype=np.float32, flags="C_CONTIGUOUS")
_i8p = np.ctypeslib.ndpointer(dtype=np.int8, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_I = ctypes.c_int64


def build() -> str:
    path = os.path.join(_HERE, "liboracle.so")
    src = os.path.join(_HERE, "tb_oracle.c")
    if not os.path.exists(path) or os.path.getmtime(path) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return path


def lib():
    global _LIB
    if _LIB is None:
        L = ctypes.CDLL(build())
        L.orc_pool_block_means.argtypes = [_f32p, _I, _I, _I, _I, _f32p]
        L.orc_kmean.argtypes = [_f32p, _I, _I, _I, _f32p]
        L.orc_quant_token_blocks.argtypes = [_f32p, _I, _I, _I, _I, _i8p, _f32p]
        L.orc_quant_k.argtypes = [_f32p, _f32p, _I, _I, _I, _I, _f32p, _i8p, _f32p]
        L.orc_block_scores.argtypes = [_f32p, _f32p, _I, _I, _I, _I, _f32p]
        L.orc_topk_from_scores.argtypes = [_f32p, _I, _I, _I, _i64p]
        L.orc_topk.argtypes = [_f32p, _f32p, _I, _I, _I, _I, _I, _i64p]
        L.orc_quantize_blockwise.argtypes = [_f32p, _I, _I, _I, _i8p, _f32p]
        L.orc_quantize_blockwise.restype = ctypes.c_int
        L.orc_w8a8.argtypes = [_i8p, _f32p, _i8p, _f32p, _I, _I, _I, _I, _f32p]
        L.orc_feature_map.argtypes = [_f32p, _I, _f32p]
        _LIB = L
    return _LIB


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def nblocks(n: int, block: int) -> int:
    return -(-n // block)


# ------------------------------------------------------------ exact parts

def pool_block_means(x, block):
    """attention.py:256-266."""
    x = _f32(x)
    h, s, d = x.shape
    out = np.empty((h, nblocks(s, block), d), np.float32)
    lib().orc_pool_block_means(x, h, s, d, block, out)
    return out


def k_mean(k):
    """attention.py:187 (sequential f32 chain over tokens)."""
    k = _f32(k)
    h, s, d = k.shape
    out = np.empty((h, d), np.float32)
    lib().orc_kmean(k, h, s, d, out)
    return out


def smooth_keys(k):
    """attention.py:179-188 -> (kc, k_mean)."""
    k = _f32(k)
    km = k_mean(k)
    return (k - km[:, None, :]).astype(np.float32), km


def quant_token_blocks(x, block):
    """attention.py:201-220 -> (codes int8 [h,s,d], scales f32 [h,nb])."""
    x = _f32(x)
    h, s, d = x.shape
    codes = np.empty((h, s, d), np.int8)
    scales = np.empty((h, nblocks(s, block)), np.float32)
    lib().orc_quant_token_blocks(x, h, s, d, block, codes, scales)
    return codes, scales


def topk_count(ratio: float, nkv: int) -> int:
    """attention.py:279 (IEEE double product, then ceil)."""
    return math.ceil(ratio * nkv)


def block_scores(qp, kp):
    qp, kp = _f32(qp), _f32(kp)
    h, nq, d = qp.shape
    nkv = kp.shape[1]
    out = np.empty((h, nq, nkv), np.float32)
    lib().orc_block_scores(qp, kp, h, nq, nkv, d, out)
    return out


def select_topk(qp, kp, ratio):
    """attention.py:269-284 -> int64 [h, nq, count], ascending per row."""
    qp, kp = _f32(qp), _f32(kp)
    h, nq, d = qp.shape
    nkv = kp.shape[1]
    count = topk_count(ratio, nkv)
    idx = np.empty((h, nq, count), np.int64)
    lib().orc_topk(qp, kp, h, nq, nkv, d, count, idx)
    return idx


def coverage(idx, nkv):
    """attention.py:114-120."""
    h, nq, c = idx.shape
    cov = np.zeros((h, nq, nkv), bool)
    if c:
        np.put_along_axis(cov, idx, True, axis=-1)
    return cov


def complement(idx, nkv):
    """attention.py:122-132: uncovered indices, ascending."""
    cov = coverage(idx, nkv)
    m = nkv - idx.shape[2]
    return np.argsort(cov, axis=-1, kind="stable")[..., :m].astype(np.int64)


def quantize_blockwise(m, block=128):
    """blockquant.py:91-110 -> (q int8, scales f32)."""
    m = _f32(m)
    if m.ndim != 2:
        raise ValueError(f"expected a matrix, got shape {m.shape}")
    r, c = m.shape
    q = np.empty((r, c), np.int8)
    sc = np.empty((nblocks(r, block), nblocks(c, block)), np.float32)
    if lib().orc_quantize_blockwise(m, r, c, block, q, sc) != 0:
        raise ValueError("input contains non-finite values")
    return q, sc


def dequantize_blockwise(q, scales, block):
    """blockquant.py:113-116."""
    r, c = q.shape
    rs = np.repeat(scales, [min(block, r - i * block) for i in range(nblocks(r, block))], axis=0)
    full = np.repeat(rs, [min(block, c - j * block) for j in range(nblocks(c, block))], axis=1)
    return q.astype(np.float32) * full


def w8a8(aq, a_scales, bq, b_scales, block):
    """blockquant.py:132-161 (exact segments, ascending k-block f32 sum)."""
    M, K = aq.shape
    N = bq.shape[1]
    out = np.empty((M, N), np.float32)
    lib().orc_w8a8(np.ascontiguousarray(aq), _f32(a_scales), np.ascontiguousarray(bq),
                   _f32(b_scales), M, K, N, block, out)
    return out


def w8a8_blas(aq, a_scales, bq, b_scales, block):
    """blockquant.py:132-161 exactly as the reference computes it for block <=
    1040: per k-block an f32 sgemm of the codes (exact: every partial sum
    stays below 2^24), ``seg *= row_scale`` then ``seg *= col_scale`` (numpy
    RN multiplies), ``out += seg`` ascending.  Same values as ``w8a8`` (the C
    restatement; tests/test_oracle_golden.py); this one runs at BLAS speed and
    is what bench.py times as the CPU baseline of configs[1]."""
    if block > 1040:
        return w8a8(aq, a_scales, bq, b_scales, block)
    M, K = aq.shape
    N = bq.shape[1]
    a32, b32 = aq.astype(np.float32), bq.astype(np.float32)
    a_s, b_s = _f32(a_scales), _f32(b_scales)
    rext = [min(block, M - i * block) for i in range(nblocks(M, block))]
    cext = [min(block, N - j * block) for j in range(nblocks(N, block))]
    out = np.zeros((M, N), np.float32)
    for kb in range(nblocks(K, block)):
        lo, hi = kb * block, min(kb * block + block, K)
        seg = a32[:, lo:hi] @ b32[lo:hi]
        np.multiply(seg, np.repeat(a_s[:, kb], rext)[:, None], out=seg)
        np.multiply(seg, np.repeat(b_s[kb], cext)[None, :], out=seg)
        out += seg
    return out


def quantized_linear(x, wq, w_scales, block=128, bias=None):
    """blockquant.py:164-182."""
    xq, xs = quantize_blockwise(x, block)
    y = w8a8(xq, xs, wq, w_scales, block)
    if bias is not None:
        y = y + _f32(bias)
    return y


# ------------------------------------------------------------ FP8 (a17)
# No reference function (the north star's "P/V to FP8");
# the rule restated here is the product's definition, pinned against
# torch's CPU float8_e4m3fn cast (tests/test_oracle_golden.py).

def e4m3_encode(x):
    """f32 -> e4m3 codes (uint8): round to nearest even, saturating to +-448
    (cvt.rn.satfinite.e4m3x2.f32); NaN -> 0x7F."""
    x = _f32(x)
    ax = np.abs(x).astype(np.float64)
    sign = np.signbit(x).astype(np.uint8) << 7
    with np.errstate(divide="ignore", invalid="ignore"):
        e = np.floor(np.log2(np.where(ax > 0, ax, 1.0)))
    e = np.clip(e, -6, 8)                             # subnormals share the 2^-6 binade's quantum 2^-9
    # exact for f32 inputs: scaling by a power of two, then rint (half-even)
    m = np.rint(ax / np.exp2(e - 3))
    e = np.where(m >= 16, e + 1, e)
    m = np.where(m >= 16, m / 2, m)                   # 16 -> next binade's 8 (exact)
    code = np.where(m >= 8, ((e + 7) * 8 + (m - 8)), m)   # m < 8 only in the subnormal binade (e = -6)
    code = np.minimum(code, 126)                      # satfinite: 0x7E = 448
    code = code.astype(np.uint8) | sign
    return np.where(np.isnan(x), np.uint8(0x7F), code).astype(np.uint8)


def e4m3_decode(c):
    c = np.asarray(c, np.uint8)
    e = ((c >> 3) & 0xF).astype(np.int32)
    m = (c & 7).astype(np.float64)
    v = np.where(e == 0, m * 2.0 ** -9, (8 + m) * np.exp2(e - 10.0))
    v = np.where((c & 0x7F) == 0x7F, np.nan, v)
    return np.where(c & 0x80, -v, v).astype(np.float32)


def quantize_v_fp8(v):
    """V [h,s,d] -> (e4m3 codes uint8 [h,s,d], per-head scales f32 [h]):
    scale = f32(absmax) / 448 (f32 RN), codes = e4m3(v / safe), safe = 1 for
    an all-zero head (the tb_quant_v_fp8 rule)."""
    v = _f32(v)
    am = np.abs(v).reshape(v.shape[0], -1).max(axis=1).astype(np.float32)
    sc = (am / np.float32(448.0)).astype(np.float32)
    safe = np.where(sc == 0, np.float32(1.0), sc).astype(np.float32)
    return e4m3_encode((v / safe[:, None, None]).astype(np.float32)), sc


# ------------------------------------------------------- float branches

def feature_map(x):
    """attention.py:287-290."""
    x = _f32(x)
    return np.where(x >= 0, x + np.float32(1), np.exp(np.minimum(x, np.float32(0)))).astype(np.float32)


def reference_attention(q, k, v, scale=None):
    """attention.py:161-176 (dense softmax, normalised after PV)."""
    q, k, v = _f32(q), _f32(k), _f32(v)
    scale = np.float32(1.0 / math.sqrt(q.shape[2]) if scale is None else scale)
    lg = scale * np.matmul(q, k.transpose(0, 2, 1))
    e = np.exp(lg - lg.max(axis=-1, keepdims=True))
    return np.matmul(e, v) / e.sum(axis=-1, keepdims=True)


def _positions(blocks, s, kvb):
    return np.concatenate([np.arange(b * kvb, min(b * kvb + kvb, s)) for b in blocks]) \
        if len(blocks) else np.empty(0, np.int64)


def sparse_branch(q, k, v, idx, qb, kvb, scale=None, quantized=True, pv_fp8=False):
    """attention.py:347-389 -> (num [h,s,d], den [h,s], row_max [h,s]).
    pv_fp8: the a17 simulation -- P (against the exact row max) and V
    (quantize_v_fp8) rounded to e4m3 for the numerator, den from f32 P."""
    q, k, v = _f32(q), _f32(k), _f32(v)
    if pv_fp8:
        vc, vs = quantize_v_fp8(v)
        vq = e4m3_decode(vc) * vs[:, None, None]
    h, s, d = q.shape
    scale = np.float32(1.0 / math.sqrt(d) if scale is None else scale)
    if quantized:
        kc, km = smooth_keys(k)
        qc, sq = quant_token_blocks(q, qb)
        kcodes, sk = quant_token_blocks(kc, kvb)
        qc32, kc32 = qc.astype(np.float32), kcodes.astype(np.float32)
    num = np.empty((h, s, d), np.float32)
    den = np.empty((h, s), np.float32)
    rmax = np.empty((h, s), np.float32)
    for hh in range(h):
        for n in range(nblocks(s, qb)):
            lo, hi = n * qb, min(n * qb + qb, s)
            blocks = idx[hh, n]
            pos = _positions(blocks, s, kvb)
            if quantized:
                ext = np.minimum(blocks * kvb + kvb, s) - blocks * kvb
                skp = np.repeat(sk[hh, blocks], ext)
                prod = qc32[hh, lo:hi] @ kc32[hh, pos].T
                corr = q[hh, lo:hi] @ km[hh]
                lg = scale * (prod * sq[hh, n] * skp[None, :] + corr[:, None])
            else:
                lg = scale * (q[hh, lo:hi] @ k[hh, pos].T)
            m = lg.max(axis=1)
            e = np.exp(lg - m[:, None])
            num[hh, lo:hi] = (e4m3_decode(e4m3_encode(e)) @ vq[hh, pos]) if pv_fp8 else e @ v[hh, pos]
            den[hh, lo:hi] = e.sum(axis=1)
            rmax[hh, lo:hi] = m
    return num, den, rmax


def linear_attention(q, k, v, comp_idx, qb, kvb):
    """attention.py:293-335 over the complement blocks -> (num, den)."""
    q, k, v = _f32(q), _f32(k), _f32(v)
    h, s, d = q.shape
    pq, pk = feature_map(q), feature_map(k)
    nkv = nblocks(s, kvb)
    kvp = np.empty((h, nkv, d, d), np.float32)
    k1p = np.empty((h, nkv, d), np.float32)
    for b in range(nkv):
        lo, hi = b * kvb, min(b * kvb + kvb, s)
        kvp[:, b] = pk[:, lo:hi].transpose(0, 2, 1) @ v[:, lo:hi]
        k1p[:, b] = pk[:, lo:hi].sum(axis=1)
    cov = coverage(comp_idx, nkv).astype(np.float32)
    kv_sel = (cov @ kvp.reshape(h, nkv, d * d)).reshape(h, -1, d, d)
    k1_sel = cov @ k1p
    num = np.empty((h, s, d), np.float32)
    den = np.empty((h, s), np.float32)
    for n in range(nblocks(s, qb)):
        lo, hi = n * qb, min(n * qb + qb, s)
        num[:, lo:hi] = pq[:, lo:hi] @ kv_sel[:, n]
        den[:, lo:hi] = (pq[:, lo:hi] @ k1_sel[:, n, :, None])[..., 0]
    return num, den


def combine(num_s, den_s, rmax, num_l, den_l, mix):
    """attention.py:416-421: shared stable normalisation."""
    ref = np.maximum(rmax, np.float32(0))
    ss = np.exp(rmax - ref)
    shrink = np.exp(-ref) * np.float32(mix)
    return (num_s * ss[..., None] + shrink[..., None] * num_l) / (den_s * ss + shrink * den_l)[..., None]


def sla_attention(q, k, v, q_block=64, kv_block=64, topk_ratio=0.1, linear_mix=1.0,
                  quantized=True, scale=None, return_parts=False, pv_fp8=False):
    """attention.py:392-421."""
    q, k, v = _f32(q), _f32(k), _f32(v)
    s = q.shape[1]
    if q_block > s or kv_block > s:
        raise ValueError(f"block sizes {q_block}/{kv_block} exceed seq {s}")
    qp, kp = pool_block_means(q, q_block), pool_block_means(k, kv_block)
    idx = select_topk(qp, kp, topk_ratio)
    nkv = kp.shape[1]
    num_s, den_s, rmax = sparse_branch(q, k, v, idx, q_block, kv_block, scale, quantized, pv_fp8)
    comp = complement(idx, nkv)
    if comp.shape[2] == 0 or linear_mix == 0.0:
        out = num_s / den_s[..., None]
    else:
        num_l, den_l = linear_attention(q, k, v, comp, q_block, kv_block)
        out = combine(num_s, den_s, rmax, num_l, den_l, linear_mix)
    if return_parts:
        return out, dict(qp=qp, kp=kp, idx=idx)
    return out


def quantized_attention(q, k, v, token_block=64, smooth_k=True, scale=None):
    """attention.py:230-253 (dense INT8 Sage attention)."""
    q, k, v = _f32(q), _f32(k), _f32(v)
    h, s, d = q.shape
    scale = np.float32(1.0 / math.sqrt(d) if scale is None else scale)
    if smooth_k:
        kc, km = smooth_keys(k)
    else:
        kc, km = k, np.zeros((h, d), np.float32)
    qc, sq = quant_token_blocks(q, token_block)
    kq, sk = quant_token_blocks(kc, token_block)
    prod = qc.astype(np.float32) @ kq.astype(np.float32).transpose(0, 2, 1)
    ext = [min(token_block, s - i * token_block) for i in range(nblocks(s, token_block))]
    sqf, skf = np.repeat(sq, ext, axis=1), np.repeat(sk, ext, axis=1)
    lg = scale * (prod * sqf[:, :, None] * skf[:, None, :] + q @ km[:, :, None])
    p = np.exp(lg - lg.max(-1, keepdims=True))
    p /= p.sum(-1, keepdims=True)
    return p @ v


def error_metrics(a, b):
    """attention.py:482-495 plus rel-L1 (north-star metric)."""
    a = np.asarray(a, np.float32).ravel().astype(np.float64)
    b = np.asarray(b, np.float32).ravel().astype(np.float64)
    daa, dbb = float(a @ a), float(b @ b)
    cos = float(a @ b / math.sqrt(daa * dbb))
    rel_l2 = float(np.linalg.norm(a - b) / math.sqrt(dbb))
    rel_l1 = float(np.abs(a - b).sum() / np.abs(b).sum())
    return cos, rel_l2, rel_l1


# ----------------------------------------------------------- sampler

def rmsnorm(x, gain, eps=1e-6):
    """sampler.py:34-40."""
    x = _f32(x)
    ms = np.mean(np.square(x), axis=-1, keepdims=True)
    return x / np.sqrt(ms + np.float32(eps)) * _f32(gain)


def layernorm(x, gain, offset, eps=1e-6):
    """sampler.py:43-52."""
    x = _f32(x)
    mu = x.mean(axis=-1, keepdims=True)
    var = np.mean(np.square(x - mu), axis=-1, keepdims=True)
    return (x - mu) / np.sqrt(var + np.float32(eps)) * _f32(gain) + _f32(offset)


def gelu(x):
    """sampler.py:55-58 (tanh approximation)."""
    c = np.float32(math.sqrt(2.0 / math.pi))
    return np.float32(0.5) * x * (np.float32(1) + np.tanh(c * (x + np.float32(0.044715) * x * x * x)))


def step_noise(seed, step, shape):
    """sampler.py:116-123."""
    return np.random.default_rng([int(seed), int(step)]).standard_normal(shape, dtype=np.float32)


def make_schedule(num_steps, sigma_max=80.0, sigma_min=0.5):
    """sampler.py:103-113."""
    lv = np.array([sigma_max]) if num_steps == 1 else np.geomspace(sigma_max, sigma_min, num_steps)
    return np.append(lv, 0.0).astype(np.float32)


def toy_block(x, sigma, w, heads, sla=None):
    """sampler.py:132-186 with quantized weights (dict of (q, scales)) and
    SLA attention (sla = dict of sla_attention kwargs) or dense attention."""
    x = _f32(x)
    seq, dim = x.shape
    hd = dim // heads
    x = x + np.float32(sigma) * w["sigma_emb"]

    def lin(a, name):
        q, sc = w[name]
        return quantized_linear(a, q, sc, 128)

    a = rmsnorm(x, w["rms_gain"])
    qkv = lin(a, "qkv")
    q, k, v = (m.reshape(seq, heads, hd).transpose(1, 0, 2) for m in np.split(qkv, 3, axis=1))
    o = sla_attention(q, k, v, **sla) if sla is not None else reference_attention(q, k, v)
    o = o.transpose(1, 0, 2).reshape(seq, dim)
    x = x + lin(o, "out_proj")
    b = layernorm(x, w["ln_gain"], w["ln_offset"])
    return x + lin(gelu(lin(b, "mlp_in")), "mlp_out")


def consistency_sample(model, sigmas, shape, seed):
    """sampler.py:281-302."""
    x = np.float32(sigmas[0]) * step_noise(seed, 0, shape)
    for i in range(len(sigmas) - 1):
        x0 = model(x, float(sigmas[i]))
        if sigmas[i + 1] > 0:
            x = x0 + np.float32(sigmas[i + 1]) * step_noise(seed, i + 1, shape)
        else:
            return x0
    return x0
