"""q_block 64 -- the reference's default SLAConfig / QuantAttnConfig block size
(attention.py:76,86-87) -- on the tcgen05 attention kernel.

The kernel runs 128-row tiles of two 64-row q-blocks over the union of their
top-k lists (tb_pair_union) and zeroes P for the rows whose q-block did not
select a block.  Checked here:
* tb_pair_union against a numpy restatement (ragged pair counts, odd nq);
* the default configurations land on the tcgen05 kernel (tb_sla_path);
* outputs against the oracle (cos >= 0.999, rel-L1 <= 1e-2) on Gaussian and
  block-coherent inputs, linear_mix 1 and 0, bf16 and f32 inputs, ragged
  lengths (last q-block and last kv-block partial, odd q-block counts);
* the exact-max instantiation's row_max / den against the oracle's sparse
  branch (attention.py:385-389), FP8 P/V and the int8 out-projection operand
  at q_block 64, and the drop-in quantized_attention (token_block 64).
"""
import numpy as np
import pytest
import torch

import gen
from oracle import oracle as O

pytestmark = pytest.mark.gpu

COS_MIN, REL_L1_MAX = 0.999, 1e-2


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


def check(got, want, what, rel=REL_L1_MAX):
    cos, _, rel1 = O.error_metrics(np.asarray(got, np.float32), np.asarray(want, np.float32))
    assert cos >= COS_MIN and rel1 <= rel, (what, cos, rel1)


def union_ref(idx):
    H, nq, count = idx.shape
    nt = -(-nq // 2)
    out, cnt = [], np.zeros((H, nt), np.int64)
    for h in range(H):
        row = []
        for t in range(nt):
            a = set(idx[h, 2 * t].tolist())
            b = set(idx[h, 2 * t + 1].tolist()) if 2 * t + 1 < nq else set()
            ent = [x | ((int(x in a) | (int(x in b) << 1)) << 28) for x in sorted(a | b)]
            cnt[h, t] = len(ent)
            row.append(ent)
        out.append(row)
    return out, cnt


@pytest.mark.parametrize("H,nq,nkv,count", [(2, 7, 40, 5), (3, 64, 64, 7), (1, 9, 1182, 119), (2, 4, 10, 10)])
def test_pair_union_matches_numpy(tb, H, nq, nkv, count):
    rng = np.random.default_rng(H * 100 + nq)
    idx = np.stack([np.stack([np.sort(rng.choice(nkv, count, replace=False)) for _ in range(nq)])
                    for _ in range(H)]).astype(np.int32)
    if nq >= 4:
        idx[0, 2] = idx[0, 3]                      # identical pair: every entry carries both bits
    pidx, pcnt = tb.pair_union(torch.from_numpy(idx).cuda())
    want, wcnt = union_ref(idx)
    pidx, pcnt = pidx.cpu().numpy(), pcnt.cpu().numpy()
    assert np.array_equal(pcnt, wcnt)
    for h in range(H):
        for t in range(pcnt.shape[1]):
            assert pidx[h, t, :pcnt[h, t]].tolist() == want[h][t], (h, t)


def test_default_configs_run_on_tensor_cores(tb):
    """SLAConfig() (64/64) and QuantAttnConfig() (token_block 64) at d = 128."""
    from paper_2512_16093_b200.attention import AttnInputs, QuantAttnConfig, quantized_attention
    q, k, v = gen.gaussian_qkv(30, 2, 1000, 128, bf16=True)
    tb.sla_attention(dev(q, True), dev(k, True), dev(v, True))          # defaults: q_block 64, kv_block 64
    assert tb.LAST_SLA_PATH == "tcgen05"
    tb.sla_attention(dev(q), dev(k), dev(v))                            # f32 inputs
    assert tb.LAST_SLA_PATH == "tcgen05"
    got = quantized_attention(AttnInputs(q, k, v), QuantAttnConfig())
    want = O.quantized_attention(q, k, v, 64, True)
    check(got, want, "quantized_attention token_block 64")


@pytest.mark.parametrize("L", [640, 1000, 4096, 4160])
@pytest.mark.parametrize("g", ["G", "B"])
@pytest.mark.parametrize("mix", [1.0, 0.0])
def test_sla_q64_vs_oracle(tb, L, g, mix):
    """L = 640 (nq 10, even) / 1000 (nq 16, ragged 40-row last q-block) / 4096 /
    4160 (nq 65: the last tile holds one q-block)."""
    q, k, v = (gen.gaussian_qkv(31, 2, L, 128, bf16=True) if g == "G"
               else gen.block_coherent_qkv(32, 2, L, 128, blk=64, bf16=True))
    want = O.sla_attention(q, k, v, 64, 64, 0.1, mix)
    for bf in (True, False):
        got = tb.sla_attention(dev(q, bf), dev(k, bf), dev(v, bf), 64, 64, 0.1, mix)
        assert tb.LAST_SLA_PATH == "tcgen05"
        check(got.cpu().numpy(), want, (L, g, mix, bf))
    gb = tb.sla_attention(dev(q, True), dev(k, True), dev(v, True), 64, 64, 0.1, mix, out_dtype=torch.bfloat16)
    check(gb.float().cpu().numpy(), want, (L, g, mix, "bf16 out"))


@pytest.mark.parametrize("ratio", [0.05, 0.3, 0.6, 1.0])
def test_sla_q64_ratios(tb, ratio):
    """Union sizes from ~count to 2*count and the all-selected case."""
    q, k, v = gen.gaussian_qkv(33, 2, 2000, 128, bf16=True)
    for mix in (1.0, 0.0):
        want = O.sla_attention(q, k, v, 64, 64, ratio, mix)
        got = tb.sla_attention(dev(q, True), dev(k, True), dev(v, True), 64, 64, ratio, mix)
        check(got.cpu().numpy(), want, (ratio, mix))


def test_sla_q64_exact_parts(tb):
    """return_parts: the exact-max instantiation with the end-of-kernel linear
    branch (two per-half numerator MMAs) and row_max / den against the
    oracle's sparse branch."""
    q, k, v = gen.gaussian_qkv(34, 2, 1000, 128, bf16=True)
    out, parts = tb.sla_attention(dev(q, True), dev(k, True), dev(v, True), 64, 64, 0.1, 1.0, return_parts=True)
    assert tb.LAST_SLA_PATH == "tcgen05"
    want = O.sla_attention(q, k, v, 64, 64, 0.1, 1.0)
    check(out.cpu().numpy(), want, "exact out")
    idx = parts["idx"].cpu().numpy().astype(np.int64)
    num, den, rmax = O.sparse_branch(q, k, v, idx, 64, 64)
    assert np.allclose(parts["row_max"].cpu().numpy(), rmax, rtol=1e-5, atol=1e-4)
    check(parts["den"].cpu().numpy(), den, "den")


def test_sla_q64_fp8_and_int8_output(tb):
    q, k, v = gen.gaussian_qkv(35, 2, 1024, 128, bf16=True)
    dq, dk, dv = dev(q, True), dev(k, True), dev(v, True)
    want = O.sla_attention(q, k, v, 64, 64, 0.1, 1.0)
    got = tb.sla_attention(dq, dk, dv, 64, 64, 0.1, 1.0, pv_fp8=True)
    assert tb.LAST_SLA_PATH == "tcgen05"
    check(got.cpu().numpy(), want, "fp8 p/v")
    ob = tb.sla_attention(dq, dk, dv, 64, 64, 0.1, 1.0, out_dtype=torch.bfloat16)
    codes, scales = tb.sla_attention(dq, dk, dv, 64, 64, 0.1, 1.0, out_dtype=torch.int8)
    wc, ws = tb.quantize_blockwise_planar(ob)
    assert torch.equal(codes, wc) and torch.equal(scales, ws)


def test_dropin_defaults_numpy(tb):
    """The drop-in with the reference's default SLAConfig on numpy inputs."""
    from paper_2512_16093_b200.attention import AttnInputs, SLAConfig, sla_attention
    q, k, v = gen.gaussian_qkv(36, 3, 2048, 128, bf16=False)
    got = sla_attention(AttnInputs(q, k, v), SLAConfig())
    want = O.sla_attention(q, k, v, 64, 64, 0.1, 1.0)
    check(got, want, "drop-in defaults")


def test_q64_union_beyond_1024_blocks(tb):
    """topk_ratio 1.0 at L = 66000 (nkv 1032): every tile walks all 1032 blocks
    (the union table holds up to 2048 entries per tile)."""
    q, k, v = gen.gaussian_qkv(37, 1, 66000, 128, bf16=True)
    got = tb.sla_attention(dev(q, True), dev(k, True), dev(v, True), 64, 64, 1.0, 1.0)
    assert tb.LAST_SLA_PATH == "tcgen05"
    want = O.sla_attention(q, k, v, 64, 64, 1.0, 1.0)
    check(got.cpu().numpy(), want, "q64 all blocks, L 66000")
