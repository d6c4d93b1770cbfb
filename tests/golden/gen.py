"""Seeded input generators shared by the golden-vector script and the tests.

Generator G: numpy default_rng Gaussian, optionally rounded
to bf16 with round-to-nearest-even so the GPU receives bf16 and the oracle
its exact f32 upcast.  Generator B: the block-coherent recipe of
/root/reference/pkg/tests/test_attention.py:302-310 (centres x3, noise 0.3),
where attention mass is concentrated and the sparse branch dominates.
"""
from __future__ import annotations

import numpy as np


def round_bf16(x: np.ndarray) -> np.ndarray:
    """Round f32 to the nearest bf16 (ties to even), returned as f32."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    lsb = (u >> 16) & 1
    u = ((u + 0x7FFF + lsb) >> 16) << 16
    return u.astype(np.uint32).view(np.float32).reshape(x.shape)


def gaussian_qkv(seed: int, h: int, s: int, d: int, bf16: bool = True):
    rng = np.random.default_rng(seed)
    out = [rng.standard_normal((h, s, d), dtype=np.float32) for _ in range(3)]
    if bf16:
        out = [round_bf16(t) for t in out]
    return out


def block_coherent_qkv(seed: int, h: int, s: int, d: int, blk: int = 64, bf16: bool = True):
    rng = np.random.default_rng(seed)
    nb = -(-s // blk)
    centers = (3.0 * rng.standard_normal((h, nb, d))).astype(np.float32)
    k = np.repeat(centers, blk, axis=1)[:, :s] + 0.3 * rng.standard_normal((h, s, d)).astype(np.float32)
    target = np.repeat(rng.integers(0, nb, (h, nb)), blk, axis=1)[:, :s]
    q = centers[np.arange(h)[:, None], target] + 0.3 * rng.standard_normal((h, s, d)).astype(np.float32)
    v = rng.standard_normal((h, s, d)).astype(np.float32)
    out = [np.ascontiguousarray(t, dtype=np.float32) for t in (q, k, v)]
    if bf16:
        out = [round_bf16(t) for t in out]
    return out


def make_inputs(gen: str, seed: int, h: int, s: int, d: int):
    if gen == "G":
        return gaussian_qkv(seed, h, s, d, bf16=True)
    if gen == "G32":
        return gaussian_qkv(seed, h, s, d, bf16=False)
    if gen == "B":
        return block_coherent_qkv(seed, h, s, d, bf16=True)
    raise ValueError(gen)


def gaussian_matrix(seed: int, rows: int, cols: int, scale: float = 1.0, bf16: bool = False):
    rng = np.random.default_rng(seed)
    m = (rng.standard_normal((rows, cols), dtype=np.float32) * np.float32(scale)).astype(np.float32)
    return round_bf16(m) if bf16 else m


# (name, generator, seed, heads, seq, head_dim, q_block, kv_block, topk_ratio)
ATTN_CASES = [
    ("cfg1", "G", 0, 2, 4096, 128, 64, 64, 0.1),
    ("cfg1_q128", "G", 0, 2, 4096, 128, 128, 64, 0.1),
    ("cfg3_h1", "G", 1, 1, 32760, 128, 128, 64, 0.1),
    ("cfg4_h1", "G", 2, 1, 75600, 128, 128, 64, 0.1),
    ("small_f32", "G32", 3, 2, 100, 16, 32, 32, 0.3),
    ("tiny_d8", "G32", 4, 3, 90, 8, 32, 32, 0.5),
    ("ragged_d64", "G32", 5, 1, 200, 64, 64, 64, 0.15),
    ("ragged_d128", "G", 6, 2, 1000, 128, 128, 64, 0.1),
    ("coherent", "B", 9, 4, 512, 64, 64, 64, 0.1),
    ("coherent_d128", "B", 7, 2, 2048, 128, 128, 64, 0.1),
]

# Headline-shape output goldens (one head, full length; tests/golden/headline.npz):
# (name, generator, seed, heads, seq, head_dim, q_block, kv_block, topk_ratio, linear_mix values)
HEADLINE_CASES = [
    ("cfg4_h1", "G", 2, 1, 75600, 128, 128, 64, 0.1, (1.0, 0.0)),
    ("cfg4_B_h1", "B", 13, 1, 75600, 128, 128, 64, 0.1, (1.0, 0.0)),
    ("cfg3_h1_q128", "G", 1, 1, 32760, 128, 128, 64, 0.1, (1.0, 0.0)),
    ("cfg3_h1_q64", "G", 1, 1, 32760, 128, 64, 64, 0.1, (1.0, 0.0)),
]


def headline_rows(s: int) -> np.ndarray:
    """Row subsample stored for the headline goldens: every 127th row plus the
    last 80 (cfg4's ragged last q-block of 128 has 80 rows)."""
    return np.unique(np.r_[np.arange(0, s, 127), np.arange(max(0, s - 80), s)]).astype(np.int64)


# (name, seed, rows, cols, scale, block)
QUANT_CASES = [
    ("q300x200", 8, 300, 200, 1.0, 128),
    ("q520x384", 11, 520, 384, 37.5, 128),
    ("q1000x1536", 1, 1000, 1536, 1.0, 128),
    ("q64x96_b32", 12, 64, 96, 1e-3, 32),
]

# (name, seed, M, K, N, block, with_bias)
W8A8_CASES = [
    ("w260x384x200", 21, 260, 384, 200, 128, True),
    ("w96x192x80_b64", 3, 96, 192, 80, 64, False),
    ("w256x1536x384", 5, 256, 1536, 384, 128, False),
]

# (nq, nkv, d) probes of the block-score GEMM order around OpenBLAS's
# small-matrix TN kernel threshold (M*N <= 1200, K >= 32, M*N*K <= 1e6)
SCORE_PROBES = [
    (30, 40, 32), (32, 40, 32), (20, 60, 32), (8, 8, 16), (16, 62, 128),
    (10, 10, 40), (4, 4, 33), (35, 35, 64), (34, 35, 64), (64, 64, 128),
    (1, 1182, 128), (9, 130, 128), (3, 7, 8), (12, 100, 17),
]
