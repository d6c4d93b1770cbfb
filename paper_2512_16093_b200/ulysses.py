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
[p*per, ...) with per = ceil(L/P) rounded up to a multiple of `align`.  Heads
must divide evenly (40 / {1,2,4,8}).

Quantized return path: with 128-aligned token shards every
128-token x 128-channel block of the attention output lives on one rank, so
the head-shard attention can emit the out-projection's block-quantized INT8
operand directly (codes + one scale per (128-token block, head)) and the
reverse all-to-all moves int8 codes instead of bf16 -- half the bytes, and no
quantization pass on the receiver.  Bit-identical to quantizing the gathered
bf16 output (per-block quantization commutes with the exchange).
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_size(L: int, P: int, align: int = 1) -> int:
    per = -(-L // P)
    return -(-per // align) * align


def token_bounds(L: int, P: int, rank: int, align: int = 1) -> tuple[int, int]:
    per = shard_size(L, P, align)
    lo = min(rank * per, L)
    return lo, min(lo + per, L)


def _world():
    if dist.is_available() and dist.is_initialized():
        return dist.get_world_size(), dist.get_rank()
    return 1, 0


def _pack_seq(x: torch.Tensor, P: int, per: int) -> torch.Tensor:
    """[L_p, H, d] token shard -> send buffer [P, per, H/P, d]: chunk j = my
    tokens of head group j (rows past L_p are never read by the receiver, so
    they stay unwritten)."""
    Lp, H, d = x.shape
    hp = H // P
    send = x.new_empty((P, per, hp, d))
    send[:, :Lp] = x.view(Lp, P, hp, d).permute(1, 0, 2, 3)
    return send


def _unpack_heads(recv: torch.Tensor, L: int) -> torch.Tensor:
    """recv [P, per, hp, d] (chunk i = rank i's tokens [i*per, ...)) -> [hp, L, d].
    token_bounds puts rank i's tokens at global [i*per, min((i+1)*per, L)), so
    the received buffer read as [P*per, hp, d] is the global token order (the
    last rank's padding lands past L): one copy."""
    P, per, hp, d = recv.shape
    return recv.view(P * per, hp, d)[:L].permute(1, 0, 2).contiguous()


def seq_to_heads(x: torch.Tensor, L: int, group=None, align: int = 1) -> torch.Tensor:
    """[L_p, H, d] token shard -> [H/P, L, d] head shard (one all-to-all)."""
    P = dist.get_world_size(group) if dist.is_initialized() else 1
    H = x.shape[1]
    if H % P:
        raise ValueError(f"heads {H} not divisible by world size {P}")
    if P == 1:
        return x.permute(1, 0, 2).contiguous()
    send = _pack_seq(x, P, shard_size(L, P, align))
    recv = torch.empty_like(send)
    dist.all_to_all_single(recv, send, group=group)
    return _unpack_heads(recv, L)


def heads_to_seq(o: torch.Tensor, L: int, group=None, align: int = 1) -> torch.Tensor:
    """[H/P, L, d] head shard -> [L_p, H, d] token shard (inverse all-to-all)."""
    P, rank = (dist.get_world_size(group), dist.get_rank(group)) if dist.is_initialized() else (1, 0)
    hp, _, d = o.shape
    if P == 1:
        return o.permute(1, 0, 2).contiguous()
    per = shard_size(L, P, align)
    send = o.new_empty((P, per, hp, d))
    send.view(P * per, hp, d)[:L] = o.permute(1, 0, 2)        # chunk i = rank i's tokens (one copy)
    recv = torch.empty_like(send)
    dist.all_to_all_single(recv, send, group=group)
    lo, hi = token_bounds(L, P, rank, align)
    # recv chunk j = my tokens for head group j
    return recv[:, :hi - lo].permute(1, 0, 2, 3).reshape(hi - lo, P * hp, d).contiguous()


def seq_to_heads_qkv(q, k, v, L: int, group=None, align: int = 1):
    """seq_to_heads of q, k and v with the three all-to-alls issued at once
    (async): each tensor's unpack copy runs while the next exchange is still
    on the wire."""
    P = dist.get_world_size(group) if dist.is_initialized() else 1
    H = q.shape[1]
    if H % P:
        raise ValueError(f"heads {H} not divisible by world size {P}")
    if P == 1:
        return tuple(t.permute(1, 0, 2).contiguous() for t in (q, k, v))
    per = shard_size(L, P, align)
    bufs = []
    for t in (q, k, v):
        send = _pack_seq(t, P, per)
        recv = torch.empty_like(send)
        bufs.append((send, recv, dist.all_to_all_single(recv, send, group=group, async_op=True)))
    out = []
    for send, recv, work in bufs:
        work.wait()
        out.append(_unpack_heads(recv, L))
    return tuple(out)


def ulysses_sla_attention(q_shard, k_shard, v_shard, L: int, attn_fn, group=None, align: int = 1):
    """Token-sharded q/k/v [L_p, H, d] -> attention on a head shard -> token-sharded o."""
    qh, kh, vh = seq_to_heads_qkv(q_shard, k_shard, v_shard, L, group, align)
    oh = attn_fn(qh, kh, vh)
    return heads_to_seq(oh.to(q_shard.dtype), L, group, align)


def heads_to_seq_q8(codes: torch.Tensor, scales: torch.Tensor, L: int, group=None, block: int = 128):
    """Head-shard block-quantized output -> token shard (quantized return path).

    codes [L, hp*d] int8 (token, local head*d + channel) and scales
    [ceil(L/block), hp] of this rank's heads -> codes [L_p, H*d] and scales
    [ceil(L_p/block), H] of this rank's 128-aligned token shard, all heads."""
    P, rank = (dist.get_world_size(group), dist.get_rank(group)) if dist.is_initialized() else (1, 0)
    if P == 1:
        return codes, scales
    hpd, hp = codes.shape[1], scales.shape[1]
    per = shard_size(L, P, block)
    nbp = per // block
    send = codes.new_zeros((P, per, hpd))
    send_s = scales.new_zeros((P, nbp, hp))
    for i in range(P):
        lo, hi = token_bounds(L, P, i, block)
        send[i, :hi - lo] = codes[lo:hi]
        b0, b1 = lo // block, -(-hi // block)
        send_s[i, :b1 - b0] = scales[b0:b1]
    recv, recv_s = torch.empty_like(send), torch.empty_like(send_s)
    dist.all_to_all_single(recv, send, group=group)
    dist.all_to_all_single(recv_s, send_s, group=group)
    lo, hi = token_bounds(L, P, rank, block)
    nb = -(-(hi - lo) // block)
    # chunk j = my tokens of head group j -> columns j*hp*d.. of the full row
    out = recv[:, :hi - lo].permute(1, 0, 2).reshape(hi - lo, P * hpd).contiguous()
    out_s = recv_s[:, :nb].permute(1, 0, 2).reshape(nb, P * hp).contiguous()
    return out, out_s


def ulysses_sla_attention_q8(q_shard, k_shard, v_shard, L: int, attn_q8_fn, group=None, block: int = 128):
    """Token-sharded q/k/v (128-aligned shards) -> head-shard attention emitting
    int8 codes + block scales -> token-shard out-projection operand."""
    qh, kh, vh = seq_to_heads_qkv(q_shard, k_shard, v_shard, L, group, block)
    codes, scales = attn_q8_fn(qh, kh, vh)
    return heads_to_seq_q8(codes, scales, L, group, block)


# ------------------------------------------------- fused return path (P2P)
# The head-shard attention's epilogue stores each 128-token tile's int8 codes
# and block scale straight into the token owner's buffers over NVLink (torch
# symmetric memory gives every rank the peers' buffer addresses), so the
# reverse exchange is part of the attention kernel: no send buffer, no
# all-to-all launch, and the transfer overlaps the attention tile by tile.
# A device-side barrier then makes every peer's stores visible before the
# out-projection reads them.  Reuse of the buffers by the next layer is
# ordered by that layer's forward all-to-all (a rank cannot start writing
# into a peer before the peer has joined it, which it does only after its
# out-projection in stream order).
_P2P = {}


def _p2p_buffers(per: int, H: int, d: int, group, device, block: int = 128):
    import torch.distributed._symmetric_memory as symm_mem
    g = group if group is not None else dist.group.WORLD
    key = (per, H, d, g.group_name, device.index)
    if key not in _P2P:
        codes = symm_mem.empty((per, H * d), dtype=torch.int8, device=device)
        scales = symm_mem.empty((per // block, H), dtype=torch.float32, device=device)
        hc = symm_mem.rendezvous(codes, g.group_name)
        hs = symm_mem.rendezvous(scales, g.group_name)
        cp = torch.tensor([int(x) for x in hc.buffer_ptrs], dtype=torch.int64, device=device)
        sp = torch.tensor([int(x) for x in hs.buffer_ptrs], dtype=torch.int64, device=device)
        _P2P[key] = (codes, scales, hc, cp, sp)
    return _P2P[key]


def attn_return_p2p(qh, kh, vh, L: int, attn_peer_fn, group=None, block: int = 128):
    """Head-shard attention whose int8 epilogue stores every tile into the
    token owner's symmetric-memory buffers, then the device barrier.  Returns
    this rank's codes [L_p, H*d] and scales [ceil(L_p/128), H] (views of its
    symmetric buffers, valid until the next call)."""
    P, rank = dist.get_world_size(group), dist.get_rank(group)
    hp, _, d = qh.shape
    H = hp * P
    per = shard_size(L, P, block)
    codes, scales, hc, cp, sp = _p2p_buffers(per, H, d, group, qh.device, block)
    attn_peer_fn(qh, kh, vh, dict(codes=cp, scales=sp, rows=per, head0=rank * hp, heads=H))
    hc.barrier()                    # all peers' tile stores into this rank's buffers are done
    lo, hi = token_bounds(L, P, rank, block)
    return codes[:hi - lo], scales[:-(-(hi - lo) // block)]


_QKV = {}


def qkv_to_heads_p2p(a_q, a_s, w_bt, w_scales, L: int, heads: int, group=None, block: int = 128):
    """Fused forward exchange: the qkv projection of this rank's (128-aligned)
    token shard with its epilogue storing every tile into the head owner's
    symmetric-memory buffer [3*hp, L, 128] (tb_w8a8_gemm_qkv_peers), then the
    device barrier.  Returns this rank's head-major q, k, v [hp, L, 128]
    (views of its buffer, valid until the next call)."""
    import torch.distributed._symmetric_memory as symm_mem
    from . import ops
    P, rank = dist.get_world_size(group), dist.get_rank(group)
    if heads % P:
        raise ValueError(f"heads {heads} not divisible by world size {P}")
    hp = heads // P
    g = group if group is not None else dist.group.WORLD
    dev = a_q.device
    key = (L, heads, g.group_name, dev.index)
    if key not in _QKV:
        buf = symm_mem.empty((3 * hp, L, 128), dtype=torch.bfloat16, device=dev)
        hdl = symm_mem.rendezvous(buf, g.group_name)
        _QKV[key] = (buf, hdl, [int(x) for x in hdl.buffer_ptrs])
    buf, hdl, ptrs = _QKV[key]
    lo, hi = token_bounds(L, P, rank, block)
    if hi - lo >= 256:
        ops.w8a8_gemm_qkv_peers(a_q, a_s, w_bt, w_scales, ptrs, heads, lo, L, block)
    elif hi > lo:
        # shard below the 2-SM kernel's 256 rows: local planes, then copies
        # into the owners' buffers through their symmetric-memory views
        planes = ops.w8a8_gemm_ex(a_q, a_s, w_bt, w_scales, block, None, torch.bfloat16, plane=128)
        for o in range(P):
            view = hdl.get_buffer(o, (3 * hp, L, 128), torch.bfloat16)
            for w in range(3):
                view[w * hp:(w + 1) * hp, lo:hi] = planes[w * heads + o * hp:w * heads + (o + 1) * hp]
    hdl.barrier()                   # every rank's q/k/v tiles are in place
    return buf[:hp], buf[hp:2 * hp], buf[2 * hp:]


def ulysses_sla_attention_q8_p2p(q_shard, k_shard, v_shard, L: int, attn_peer_fn, group=None, block: int = 128):
    """ulysses_sla_attention_q8 with the reverse exchange fused into the
    attention epilogue (peer-memory stores).  attn_peer_fn(qh, kh, vh,
    peer_out) runs the head-shard attention with ops.sla_attention(...,
    out_dtype=torch.int8, peer_out=peer_out)."""
    P = dist.get_world_size(group)
    if q_shard.shape[1] % P:
        raise ValueError(f"heads {q_shard.shape[1]} not divisible by world size {P}")
    qh, kh, vh = seq_to_heads_qkv(q_shard, k_shard, v_shard, L, group, block)
    return attn_return_p2p(qh, kh, vh, L, attn_peer_fn, group, block)
