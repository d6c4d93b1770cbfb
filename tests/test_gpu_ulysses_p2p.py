"""Fused Ulysses return path (tb_sla_args.out_peers): the attention epilogue
stores every 128-token tile of the int8 out-projection operand straight into
the token owner's buffers.  One GPU emulates P ranks: each head group's
attention runs in turn with the P owners' buffers (all local here, peer memory
on a multi-GPU box) as targets, and every owner's buffer must equal the token
rows of the unsharded int8 output bit-for-bit."""
import numpy as np
import pytest
import torch

import gen
from paper_2512_16093_b200 import ulysses

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ops():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2512_16093_b200 import _lib, ops as o
    _lib.load(require_device=True)
    return o


@pytest.mark.parametrize("P,L,fp8", [(2, 1000, False), (4, 2100, False), (2, 1500, True)])
def test_peer_epilogue_matches_unsharded_int8_output(ops, P, L, fp8):
    H, d = 8, 128
    q, k, v = (torch.from_numpy(t).cuda().to(torch.bfloat16) for t in gen.gaussian_qkv(41, H, L, d, bf16=True))
    want_c, want_s = ops.sla_attention(q, k, v, 128, 64, 0.1, 1.0, out_dtype=torch.int8, pv_fp8=fp8)
    per = ulysses.shard_size(L, P, 128)
    codes = [torch.full((per, H * d), 77, dtype=torch.int8, device="cuda") for _ in range(P)]
    scales = [torch.full((per // 128, H), -1.0, device="cuda") for _ in range(P)]
    cp = torch.tensor([c.data_ptr() for c in codes], dtype=torch.int64, device="cuda")
    sp = torch.tensor([s.data_ptr() for s in scales], dtype=torch.int64, device="cuda")
    hp = H // P
    for g in range(P):                                  # rank g's head shard
        sl = slice(g * hp, (g + 1) * hp)
        r = ops.sla_attention(q[sl].contiguous(), k[sl].contiguous(), v[sl].contiguous(), 128, 64, 0.1, 1.0,
                              out_dtype=torch.int8, pv_fp8=fp8,
                              peer_out=dict(codes=cp, scales=sp, rows=per, head0=g * hp, heads=H))
        assert r is None
    torch.cuda.synchronize()
    for rank in range(P):
        lo, hi = ulysses.token_bounds(L, P, rank, 128)
        nb = -(-(hi - lo) // 128)
        assert torch.equal(codes[rank][:hi - lo], want_c[lo:hi]), rank
        assert torch.equal(scales[rank][:nb], want_s[lo // 128:lo // 128 + nb]), rank


def test_peer_epilogue_rejects_bad_rows(ops):
    q = torch.zeros((2, 256, 128), dtype=torch.bfloat16, device="cuda")
    z = torch.zeros(2, dtype=torch.int64, device="cuda")
    with pytest.raises(ValueError):
        ops.sla_attention(q, q, q, 128, 64, 0.1, 1.0, out_dtype=torch.int8,
                          peer_out=dict(codes=z, scales=z, rows=100, head0=0, heads=2))


def _p2p_world1(port, out_q):
    import os
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    try:
        torch.cuda.set_device(0)
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
        from paper_2512_16093_b200 import _lib, ops as o
        _lib.load(require_device=True)
        H, L, d = 4, 1000, 128
        q, k, v = (torch.from_numpy(t).cuda().to(torch.bfloat16) for t in gen.gaussian_qkv(42, H, L, d, bf16=True))
        want_c, want_s = o.sla_attention(q, k, v, 128, 64, 0.1, 1.0, out_dtype=torch.int8)
        shard = [t.permute(1, 0, 2).contiguous() for t in (q, k, v)]      # [L, H, d] token shard (P = 1)

        def attn_peer(qh, kh, vh, peer_out):
            return o.sla_attention(qh, kh, vh, 128, 64, 0.1, 1.0, out_dtype=torch.int8, peer_out=peer_out)
        c, s = ulysses.ulysses_sla_attention_q8_p2p(shard[0], shard[1], shard[2], L, attn_peer)
        torch.cuda.synchronize()
        ok = torch.equal(c, want_c) and torch.equal(s, want_s)
        # the fused forward exchange through symmetric memory (qkv GEMM epilogue)
        dim = H * d
        g = torch.Generator(device="cuda").manual_seed(6)
        x = torch.randn((L, dim), generator=g, device="cuda").to(torch.bfloat16)
        wq, ws = o.quantize_blockwise(torch.randn((dim, 3 * dim), generator=g, device="cuda") / dim ** 0.5, 128)
        bt = o.transpose_codes(wq)
        aq, asc = o.quantize_blockwise(x, 128, check_finite=False)
        planes = o.w8a8_gemm_ex(aq, asc, bt, ws, 128, None, torch.bfloat16, plane=128)
        qh, kh, vh = ulysses.qkv_to_heads_p2p(aq, asc, bt, ws, L, H)
        torch.cuda.synchronize()
        ok_qkv = torch.equal(torch.cat([qh, kh, vh]), planes)
        out_q.put((bool(ok), bool(ok_qkv), ""))
        dist.destroy_process_group()
    except Exception as e:                              # report instead of hanging the parent
        out_q.put((False, False, repr(e)))


def test_peer_memory_path_world1():
    """The real paths (IPC peer allocations, pointer tables, device barriers)
    at world size 1 on the one GPU: the attention return and the qkv forward
    exchange equal the plain outputs."""
    import socket
    import torch.multiprocessing as mp
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    ctx = mp.get_context("spawn")
    qq = ctx.Queue()
    p = ctx.Process(target=_p2p_world1, args=(port, qq))
    p.start()
    ok_attn, ok_qkv, err = qq.get(timeout=240)
    p.join(timeout=60)
    assert ok_attn and ok_qkv, (ok_attn, ok_qkv, err)


@pytest.mark.parametrize("P,L", [(2, 1000), (4, 2400)])
def test_qkv_peer_epilogue_matches_planar_gemm(ops, P, L):
    """tb_w8a8_gemm_qkv_peers: every emulated rank's qkv projection of its
    128-aligned token rows, stored into the head owners' [3*hp, L, 128]
    buffers, reassembles the unsharded head-major planes bit-for-bit."""
    H, d = 4, 128
    dim = H * d
    g = torch.Generator(device="cuda").manual_seed(5)
    x = torch.randn((L, dim), generator=g, device="cuda").to(torch.bfloat16)
    w = torch.randn((dim, 3 * dim), generator=g, device="cuda") / dim ** 0.5
    wq, ws = ops.quantize_blockwise(w, 128)
    bt = ops.transpose_codes(wq)
    aq, asc = ops.quantize_blockwise(x, 128, check_finite=False)
    planes = ops.w8a8_gemm_ex(aq, asc, bt, ws, 128, None, torch.bfloat16, plane=128)     # [3H, L, 128]
    hp = H // P
    bufs = [torch.full((3 * hp, L, 128), float("nan"), dtype=torch.bfloat16, device="cuda") for _ in range(P)]
    ptrs = [b.data_ptr() for b in bufs]
    for rank in range(P):
        lo, hi = ulysses.token_bounds(L, P, rank, 128)
        assert hi - lo >= 256
        ops.w8a8_gemm_qkv_peers(aq[lo:hi].contiguous(), asc[lo // 128:-(-hi // 128)].contiguous(), bt, ws, ptrs,
                                H, lo, L)
    torch.cuda.synchronize()
    for o in range(P):
        for wi in range(3):
            want = planes[wi * H + o * hp:wi * H + (o + 1) * hp]
            assert torch.equal(bufs[o][wi * hp:(wi + 1) * hp], want), (o, wi)
