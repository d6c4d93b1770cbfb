"""Ulysses head-parallel sharding of the SLA attention (new; the reference is
single-process).

Every hot-path quantity of SLA attention is per head (pooling, top-k,
k_mean, Q/K codes, linear branch, combine: attention.py:187,264,280,370), so
head sharding is numerically identical to one GPU.  The DiT is sequence-
parallel outside attention; the boundary is one all-to-all each way:

    q, k, v  [L/P, H, d] (token shard)  --a2a-->  [H/P, L, d] (head shard)
    o        [H/P, L, d]                --a2a-->  [L/P, H, d]

over NCCL (torch.distributed, backend "nccl"; "gloo" for CPU tests of the
index math).  Token shards may be uneven (L % P != 0): shard p owns tokens
[p*ceil(L/P), ...).  Heads must divide evenly (40 / {1,2,4,8}).
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def token_bounds(L: int, P: int, rank: int) -> tuple[int, int]:
    per = -(-L // P)
    lo = min(rank * per, L)
    return lo, min(lo + per, L)


def _world():
    if dist.is_available() and dist.is_initialized():
        return dist.get_world_size(), dist.get_rank()
    return 1, 0


def seq_to_heads(x: torch.Tensor, L: int, group=None) -> torch.Tensor:
    """[L_p, H, d] token shard -> [H/P, L, d] head shard (one all-to-all)."""
    P, rank = (dist.get_world_size(group), dist.get_rank(group)) if dist.is_initialized() else (1, 0)
    Lp, H, d = x.shape
    if H % P:
        raise ValueError(f"heads {H} not divisible by world size {P}")
    hp = H // P
    if P == 1:
        return x.permute(1, 0, 2).contiguous()
    per = -(-L // P)
    # send buffer [P, per, hp, d]: chunk j = my tokens for head group j (padded to `per` rows)
    send = x.new_zeros((P, per, hp, d))
    send[:, :Lp] = x.view(Lp, P, hp, d).permute(1, 0, 2, 3)
    recv = torch.empty_like(send)
    dist.all_to_all_single(recv, send, group=group)
    # recv chunk i = tokens of rank i for my head group
    out = x.new_empty((hp, L, d))
    for i in range(P):
        lo, hi = token_bounds(L, P, i)
        out[:, lo:hi] = recv[i, :hi - lo].permute(1, 0, 2)
    return out


def heads_to_seq(o: torch.Tensor, L: int, group=None) -> torch.Tensor:
    """[H/P, L, d] head shard -> [L_p, H, d] token shard (inverse all-to-all)."""
    P, rank = (dist.get_world_size(group), dist.get_rank(group)) if dist.is_initialized() else (1, 0)
    hp, _, d = o.shape
    if P == 1:
        return o.permute(1, 0, 2).contiguous()
    per = -(-L // P)
    send = o.new_zeros((P, per, hp, d))
    for i in range(P):
        lo, hi = token_bounds(L, P, i)
        send[i, :hi - lo] = o[:, lo:hi].permute(1, 0, 2)
    recv = torch.empty_like(send)
    dist.all_to_all_single(recv, send, group=group)
    lo, hi = token_bounds(L, P, rank)
    # recv chunk j = my tokens for head group j
    return recv[:, :hi - lo].permute(1, 0, 2, 3).reshape(hi - lo, P * hp, d).contiguous()


def ulysses_sla_attention(q_shard, k_shard, v_shard, L: int, attn_fn, group=None):
    """Token-sharded q/k/v [L_p, H, d] -> attention on a head shard -> token-sharded o."""
    qh = seq_to_heads(q_shard, L, group)
    kh = seq_to_heads(k_shard, L, group)
    vh = seq_to_heads(v_shard, L, group)
    oh = attn_fn(qh, kh, vh)
    return heads_to_seq(oh.to(q_shard.dtype), L, group)
