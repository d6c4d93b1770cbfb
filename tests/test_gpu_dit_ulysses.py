"""Sequence-parallel DiT block on one GPU with two ranks: the Ulysses exchange
(gloo, CUDA tensors staged through the host) around the real kernels, with the
quantized return path (int8 attention output codes + block scales crossing the
reverse all-to-all).  Every kernel is row- or head-local and the token shards
are 128-aligned, so the two-rank block output equals the one-rank output
bit-for-bit."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

L, DIM, HEADS, FFN = 700, 256, 2, 512
SLA = dict(q_block=128, kv_block=64, topk_ratio=0.25, linear_mix=1.0)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


class _Done:
    def wait(self):
        return True


def _staged_all_to_all(out, inp, group=None, async_op=False, **kw):
    # gloo has no CUDA all_to_all: stage through host memory (synchronously;
    # an async caller gets an already-completed work handle)
    h_out = torch.empty(out.shape, dtype=out.dtype)
    _orig_a2a(h_out, inp.cpu(), group=group)
    out.copy_(h_out)
    return _Done() if async_op else None


_orig_a2a = dist.all_to_all_single


def _block(world, rank):
    from paper_2512_16093_b200 import dit, ulysses
    layer = dit.random_layers(DIM, FFN, 1, seed=3)[0]
    g = torch.Generator(device="cuda").manual_seed(9)
    x = torch.randn((L, DIM), generator=g, device="cuda")
    lo, hi = ulysses.token_bounds(L, world, rank, dit.TOKEN_ALIGN)
    xo, pend = dit.block_forward(x[lo:hi].contiguous(), 0.7, layer, HEADS, SLA, L)
    return (xo if pend is None else xo + pend).cpu(), lo, hi


def _worker(rank, world, port, ref_path, out_q, p2p=False):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    if p2p:
        os.environ["TB_ULYSSES_P2P"] = "1"
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        dist.all_to_all_single = _staged_all_to_all
        torch.cuda.set_device(0)
        out, lo, hi = _block(world, rank)
        ref = torch.load(ref_path)
        out_q.put((rank, torch.equal(out, ref[lo:hi]), (out - ref[lo:hi]).abs().max().item()))
        dist.destroy_process_group()
    except Exception as e:                      # report instead of leaving the parent waiting
        out_q.put((rank, False, repr(e)))


@pytest.mark.gpu
@pytest.mark.parametrize("p2p", [False, True], ids=["nccl-path", "p2p"])
def test_dit_block_two_ranks_equals_one_rank(tmp_path, p2p):
    """p2p: both exchanges fused into their producers over peer memory
    (TB_ULYSSES_P2P=1) -- two processes on the one GPU, so the IPC handle
    exchange, the cross-process peer stores and the device barriers are the
    real multi-rank ones."""
    ref, _, _ = _block(1, 0)
    ref_path = str(tmp_path / "ref.pt")
    torch.save(ref, ref_path)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, ref_path, q, p2p), daemon=True) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
    for rank, same, err in res:
        assert same, (rank, err)


STEPS = 3


def _sample(world, rank):
    """Full rCM sample (sampler.py:281-302) of a 2-layer toy DiT: the initial
    state and every step's noise are the reference's (seed, step) streams
    (sampler.py:116-123, drawn for the WHOLE sequence) and each rank keeps its
    token shard, so the sharded sample must equal the one-rank sample."""
    import numpy as np
    from paper_2512_16093_b200 import dit, sampler, ulysses
    layers = dit.random_layers(DIM, FFN, 2, seed=4)
    lo, hi = ulysses.token_bounds(L, world, rank, dit.TOKEN_ALIGN)
    sig = sampler.make_schedule(STEPS).sigmas.tolist()
    eps = [torch.from_numpy(sampler.step_noise(11, i, (L, DIM))[lo:hi].copy()).cuda() for i in range(STEPS)]
    out = dit.rcm_sample(layers, HEADS, SLA, eps[0], eps[1:], sig, L_global=L)
    return out.cpu(), lo, hi


def _sample_worker(rank, world, port, ref_path, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        dist.all_to_all_single = _staged_all_to_all
        torch.cuda.set_device(0)
        out, lo, hi = _sample(world, rank)
        ref = torch.load(ref_path)
        out_q.put((rank, torch.equal(out, ref[lo:hi]), (out - ref[lo:hi]).abs().max().item()))
        dist.destroy_process_group()
    except Exception as e:
        out_q.put((rank, False, repr(e)))


@pytest.mark.gpu
def test_rcm_sample_two_ranks_equals_one_rank(tmp_path):
    """the sampler is replicated, each rank's noise is its token
    slice of the global (seed, step) stream -> bit-identical to one GPU."""
    ref, _, _ = _sample(1, 0)
    assert torch.isfinite(ref).all()
    ref_path = str(tmp_path / "ref_sample.pt")
    torch.save(ref, ref_path)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sample_worker, args=(r, 2, port, ref_path, q), daemon=True) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
    for rank, same, err in res:
        assert same, (rank, err)
