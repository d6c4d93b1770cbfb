"""Ulysses head-parallel sharding: index math of the all-to-all exchange, run
with world size 2 (and 4) on the CPU ``gloo`` backend.  The attention function
is a per-head stand-in, so the test checks exactly what the collective must
guarantee: head-sharded attention over token-sharded inputs equals the
unsharded computation, with uneven token shards."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2512_16093_b200 import ulysses


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def per_head_fn(q, k, v):
    # any per-head function of the full sequence (softmax attention, f64 for exactness)
    lg = torch.einsum("hld,hmd->hlm", q.double(), k.double()) / q.shape[-1] ** 0.5
    return torch.einsum("hlm,hmd->hld", torch.softmax(lg, -1), v.double()).float()


def _worker(rank, world, port, L, H, d, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = torch.Generator().manual_seed(0)
    q, k, v = (torch.randn((L, H, d), generator=g) for _ in range(3))   # global [L, H, d]
    lo, hi = ulysses.token_bounds(L, world, rank)
    # token shard -> head shard -> token shard round trip is the identity
    hs = ulysses.seq_to_heads(q[lo:hi].contiguous(), L)
    hp = H // world
    ok_heads = torch.equal(hs, q[:, rank * hp:(rank + 1) * hp].permute(1, 0, 2))
    back = ulysses.heads_to_seq(hs, L)
    ok_back = torch.equal(back, q[lo:hi])
    o = ulysses.ulysses_sla_attention(q[lo:hi].contiguous(), k[lo:hi].contiguous(), v[lo:hi].contiguous(),
                                      L, per_head_fn)
    ref = per_head_fn(q.permute(1, 0, 2), k.permute(1, 0, 2), v.permute(1, 0, 2)).permute(1, 0, 2)[lo:hi]
    err = (o - ref).abs().max().item()
    out_q.put((rank, ok_heads, ok_back, err))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,L,H", [(2, 37, 4), (2, 64, 2), (4, 50, 8)])
def test_ulysses_roundtrip_and_attention(world, L, H):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, L, H, 8, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for rank, ok_heads, ok_back, err in res:
        assert ok_heads and ok_back, rank
        assert err < 1e-5, (rank, err)


def test_token_bounds_cover_sequence():
    for L in (1, 7, 75600, 32760):
        for P in (1, 2, 4, 8):
            for align in (1, 128):
                spans = [ulysses.token_bounds(L, P, r, align) for r in range(P)]
                assert spans[0][0] == 0 and spans[-1][1] == L
                assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
                assert all(lo % align == 0 for lo, hi in spans if hi > lo)


def _worker_q8(rank, world, port, L, H, d, out_q):
    """Quantized return path: a head shard's int8 codes [L, hp*d] + block scales
    [nq, hp] arrive as this rank's 128-aligned token shard of the global
    [L, H*d] codes and [nq, H] scales; the aligned q/k/v exchange round-trips."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = torch.Generator().manual_seed(1)
    nq = -(-L // 128)
    codes = torch.randint(-127, 128, (L, H * d), generator=g, dtype=torch.int8)    # global operand
    scales = torch.rand((nq, H), generator=g)
    hp = H // world
    mine_c = codes.view(L, H, d)[:, rank * hp:(rank + 1) * hp].reshape(L, hp * d).contiguous()
    mine_s = scales[:, rank * hp:(rank + 1) * hp].contiguous()
    oc, os_ = ulysses.heads_to_seq_q8(mine_c, mine_s, L, block=128)
    lo, hi = ulysses.token_bounds(L, world, rank, 128)
    ok_c = torch.equal(oc, codes[lo:hi])
    ok_s = torch.equal(os_, scales[lo // 128: -(-hi // 128)])
    q = torch.randn((L, H, d), generator=g)
    hs = ulysses.seq_to_heads(q[lo:hi].contiguous(), L, align=128)
    ok_rt = torch.equal(ulysses.heads_to_seq(hs, L, align=128), q[lo:hi])
    out_q.put((rank, ok_c, ok_s, ok_rt))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,L,H", [(2, 300, 4), (4, 1000, 8), (2, 256, 2)])
def test_ulysses_quantized_return_path(world, L, H):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_q8, args=(r, world, port, L, H, 16, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for rank, ok_c, ok_s, ok_rt in res:
        assert ok_c and ok_s and ok_rt, rank
