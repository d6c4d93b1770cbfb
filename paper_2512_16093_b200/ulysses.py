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


# ------------------------------------------------- fused exchanges (P2P)
# Both exchanges can ride NVLink inside their producers: the qkv projection's
# epilogue stores every tile into the HEAD owner's buffer, and the attention's
# int8 epilogue stores every tile into the TOKEN owner's buffer, so a DiT layer
# needs no send buffers, no all-to-all launches and no unpack copies, and the
# transfers overlap the producing kernels tile by tile.  The buffers are
# dedicated allocations mapped into every rank's process with CUDA IPC
# (csrc/peer.cu; valid for one process per GPU over NVLink, and for several
# processes sharing a GPU, which is how the multi-rank path is tested here), and
# a stream-ordered device barrier over flag blocks in the same memory makes the
# peers' stores visible before the consumer runs.  Buffer reuse across layers is
# ordered by those barriers.


def _tensor_at(addr: int, shape, dtype, device) -> torch.Tensor:
    """Zero-copy torch view of device memory at `addr` (own or peer-mapped)."""
    elt = {torch.int8: ("|i1", 1), torch.uint8: ("|u1", 1), torch.float32: ("<f4", 4),
           torch.bfloat16: ("<i2", 2), torch.int32: ("<i4", 4)}[dtype]

    class _CAI:
        __cuda_array_interface__ = {"shape": tuple(shape), "typestr": elt[0], "data": (int(addr), False),
                                    "version": 3, "strides": None}
    t = torch.as_tensor(_CAI(), device=device)
    return t.view(torch.bfloat16) if dtype == torch.bfloat16 else t


class PeerGroup:
    """Per-process-group peer memory: allocations every rank can store into,
    and the group's device barrier.  ``alloc`` is a collective (every rank of
    the group must call it in the same order), so callers allocate at setup
    (``prepare_p2p``), not lazily inside a forward pass that ranks may take
    differently; ``close`` (also a context-manager exit) unmaps the peers'
    allocations and frees this rank's own."""

    def __init__(self, group=None):
        import ctypes
        from . import _lib
        self.ctypes, self.lib = ctypes, _lib.load(require_device=True)
        self.group = group
        self.P, self.rank = dist.get_world_size(group), dist.get_rank(group)
        self.device = torch.device("cuda", torch.cuda.current_device())
        self.epoch = 0
        self._own, self._imported = [], []
        flags = self.alloc(4 * self.P)
        self.flag_table = torch.tensor(flags, dtype=torch.int64, device=self.device)

    def alloc(self, nbytes: int) -> list[int]:
        """A zeroed allocation of nbytes on every rank -> the P addresses, as
        seen from this process (own pointer at index rank)."""
        c = self.ctypes
        p = c.c_void_p()
        _check(self.lib.tb_peer_alloc(nbytes, c.byref(p)), "tb_peer_alloc")
        self._own.append(int(p.value))
        h = c.create_string_buffer(64)
        _check(self.lib.tb_peer_export(p, h), "tb_peer_export")
        handles = [None] * self.P
        dist.all_gather_object(handles, bytes(h.raw), group=self.group)
        ptrs = []
        for r, hr in enumerate(handles):
            if r == self.rank:
                ptrs.append(int(p.value))
            else:
                q = c.c_void_p()
                _check(self.lib.tb_peer_import(c.create_string_buffer(hr, 64), c.byref(q)), "tb_peer_import")
                self._imported.append(int(q.value))
                ptrs.append(int(q.value))
        return ptrs

    def close(self):
        """Collective teardown: wait for this rank's work, meet the peers (no
        rank may still be storing into memory about to be unmapped), unmap
        the imported allocations, free the own ones."""
        if self._own is None:
            return
        torch.cuda.synchronize(self.device)
        dist.barrier(group=self.group)
        c = self.ctypes
        for q in self._imported:
            _check(self.lib.tb_peer_close(c.c_void_p(q)), "tb_peer_close")
        dist.barrier(group=self.group)      # every peer has unmapped before the owners free
        for p in self._own:
            _check(self.lib.tb_peer_free(c.c_void_p(p)), "tb_peer_free")
        self._own = self._imported = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
        return False

    def barrier(self):
        from .ops import stream_ptr
        self.epoch += 1
        _check(self.lib.tb_peer_barrier(self.ctypes.c_void_p(self.flag_table.data_ptr()), self.P, self.rank,
                                        self.epoch, stream_ptr()), "tb_peer_barrier")


def _check(rc: int, what: str):
    from . import _lib
    _lib.check(rc, what)


_GROUPS = {}


def peer_group(group=None) -> PeerGroup:
    g = group if group is not None else dist.group.WORLD
    key = (g.group_name, torch.cuda.current_device())
    if key not in _GROUPS:
        _GROUPS[key] = PeerGroup(group)
    return _GROUPS[key]


def close_peer_groups():
    """Release every peer group and the exchange buffers cached on them
    (collective over each group)."""
    for key in list(_P2P):
        del _P2P[key]
    for key in list(_QKV):
        del _QKV[key]
    for key, pg in list(_GROUPS.items()):
        pg.close()
        del _GROUPS[key]


def prepare_p2p(L: int, heads: int, d: int = 128, group=None, block: int = 128):
    """Allocate (collectively, at setup) both fused-exchange buffer sets of a
    DiT with L tokens and `heads` heads, so the forward pass never runs the
    allocation collective."""
    P = dist.get_world_size(group)
    per = shard_size(L, P, block)
    dev = torch.device("cuda", torch.cuda.current_device())
    _p2p_buffers(per, heads, d, group, dev, block)
    _qkv_buffers(L, heads, group, dev)


_P2P = {}


def _p2p_buffers(per: int, H: int, d: int, group, device, block: int = 128):
    pg = peer_group(group)
    key = (per, H, d, id(pg))
    if key not in _P2P:
        cptrs = pg.alloc(per * H * d)
        sptrs = pg.alloc(4 * (per // block) * H)
        codes = _tensor_at(cptrs[pg.rank], (per, H * d), torch.int8, device)
        scales = _tensor_at(sptrs[pg.rank], (per // block, H), torch.float32, device)
        cp = torch.tensor(cptrs, dtype=torch.int64, device=device)
        sp = torch.tensor(sptrs, dtype=torch.int64, device=device)
        _P2P[key] = (codes, scales, pg, cp, sp)
    return _P2P[key]


def attn_return_p2p(qh, kh, vh, L: int, attn_peer_fn, group=None, block: int = 128):
    """Head-shard attention whose int8 epilogue stores every tile into the
    token owner's peer buffers, then the device barrier.  Returns
    this rank's codes [L_p, H*d] and scales [ceil(L_p/128), H] (views of its
    peer buffers, valid until the next call)."""
    P, rank = dist.get_world_size(group), dist.get_rank(group)
    hp, _, d = qh.shape
    H = hp * P
    per = shard_size(L, P, block)
    codes, scales, pg, cp, sp = _p2p_buffers(per, H, d, group, qh.device, block)
    attn_peer_fn(qh, kh, vh, dict(codes=cp, scales=sp, rows=per, head0=rank * hp, heads=H))
    pg.barrier()                    # all peers' tile stores into this rank's buffers are done
    lo, hi = token_bounds(L, P, rank, block)
    return codes[:hi - lo], scales[:-(-(hi - lo) // block)]


_QKV = {}


def _qkv_buffers(L: int, heads: int, group, device):
    pg = peer_group(group)
    hp = heads // pg.P
    key = (L, heads, id(pg))
    if key not in _QKV:
        ptrs = pg.alloc(3 * hp * L * 128 * 2)
        _QKV[key] = (_tensor_at(ptrs[pg.rank], (3 * hp, L, 128), torch.bfloat16, device), ptrs, pg)
    return _QKV[key]


def qkv_to_heads_p2p(a_q, a_s, w_bt, w_scales, L: int, heads: int, group=None, block: int = 128):
    """Fused forward exchange: the qkv projection of this rank's (128-aligned)
    token shard with its epilogue storing every tile into the head owner's
    peer buffer [3*hp, L, 128] (tb_w8a8_gemm_qkv_peers), then the device
    barrier.  Returns this rank's head-major q, k, v [hp, L, 128] (views of
    its buffer, valid until the next call)."""
    from . import ops
    P, rank = dist.get_world_size(group), dist.get_rank(group)
    if heads % P:
        raise ValueError(f"heads {heads} not divisible by world size {P}")
    hp = heads // P
    dev = a_q.device
    buf, ptrs, pg = _qkv_buffers(L, heads, group, dev)
    lo, hi = token_bounds(L, P, rank, block)
    if hi - lo >= 256:
        ops.w8a8_gemm_qkv_peers(a_q, a_s, w_bt, w_scales, ptrs, heads, lo, L, block)
    elif hi > lo:
        # shard below the 2-SM kernel's 256 rows: local planes, then copies
        # into the owners' buffers through their peer-mapped views
        planes = ops.w8a8_gemm_ex(a_q, a_s, w_bt, w_scales, block, None, torch.bfloat16, plane=128)
        for o in range(P):
            view = _tensor_at(ptrs[o], (3 * hp, L, 128), torch.bfloat16, dev)
            for w in range(3):
                view[w * hp:(w + 1) * hp, lo:hi] = planes[w * heads + o * hp:w * heads + (o + 1) * hp]
    pg.barrier()                    # every rank's q/k/v tiles are in place
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


# ------------------------------------------------ C-ABI exchange (native)
# The same two exchanges as entry points of libtb200.so (csrc/ulysses.cu:
# tb_ulysses_seq_to_heads / tb_ulysses_heads_to_seq): pack,
# grouped ncclSend/ncclRecv over a caller-provided communicator, unpack -- the
# path a host that binds the C ABI (not torch.distributed) uses.  Identical
# layout to _pack_seq / _unpack_heads above.

TB_UL_PACK, TB_UL_EXCHANGE, TB_UL_UNPACK, TB_UL_ALL = 1, 2, 4, 7
_ESIZE = {torch.bfloat16: 2, torch.float16: 2, torch.float32: 4, torch.int8: 1, torch.uint8: 1}


def native_seq_to_heads(x: torch.Tensor, L: int, P: int, rank: int, align: int = 1, comm=None,
                        stages: int = TB_UL_ALL, send=None, recv=None, out=None):
    """tb_ulysses_seq_to_heads: token shard [L_p, H, d] -> head shard [H/P, L, d].
    Returns (out, send, recv) (the workspaces are returned so a caller running
    the exchange itself -- stages without TB_UL_EXCHANGE -- can fill recv)."""
    from . import _lib
    from .ops import ptr, stream_ptr
    import ctypes
    Lp, H, d = x.shape
    lib = _lib.load(require_device=True)
    per = lib.tb_ulysses_shard(L, P, align)
    if send is None:
        send = torch.empty((P, per, H // P, d), dtype=x.dtype, device=x.device)
    if recv is None:
        recv = torch.empty_like(send)
    if out is None:
        out = torch.empty((H // P, L, d), dtype=x.dtype, device=x.device)
    _check(lib.tb_ulysses_seq_to_heads(ptr(x.contiguous()), L, H, d, _ESIZE[x.dtype], P, rank, align, ptr(send),
                                       ptr(recv), ptr(out), ctypes.c_void_p(comm), stages, stream_ptr()),
           "tb_ulysses_seq_to_heads")
    return out, send, recv


def native_heads_to_seq(o: torch.Tensor, L: int, P: int, rank: int, align: int = 1, comm=None,
                        stages: int = TB_UL_ALL, send=None, recv=None, out=None):
    """tb_ulysses_heads_to_seq: head shard [H/P, L, d] -> token shard [L_p, H, d]."""
    from . import _lib
    from .ops import ptr, stream_ptr
    import ctypes
    hp, _, d = o.shape
    H = hp * P
    lib = _lib.load(require_device=True)
    per = lib.tb_ulysses_shard(L, P, align)
    lo, hi = token_bounds(L, P, rank, align)
    if send is None:
        send = torch.empty((P, per, hp, d), dtype=o.dtype, device=o.device)
    if recv is None:
        recv = torch.empty_like(send)
    if out is None:
        out = torch.empty((hi - lo, H, d), dtype=o.dtype, device=o.device)
    _check(lib.tb_ulysses_heads_to_seq(ptr(o.contiguous()), L, H, d, _ESIZE[o.dtype], P, rank, align, ptr(send),
                                       ptr(recv), ptr(out), ctypes.c_void_p(comm), stages, stream_ptr()),
           "tb_ulysses_heads_to_seq")
    return out, send, recv


class NcclComm:
    """An NCCL communicator made through the C ABI (tb_nccl_unique_id /
    tb_nccl_comm_init) for a torch.distributed group: rank 0's unique id is
    broadcast with broadcast_object_list, every rank joins.  ``handle`` is
    the raw ncclComm_t for native_seq_to_heads / native_heads_to_seq."""

    def __init__(self, group=None):
        import ctypes
        from . import _lib
        self.lib = _lib.load(require_device=True)
        self.P, self.rank = dist.get_world_size(group), dist.get_rank(group)
        uid = ctypes.create_string_buffer(128)
        if self.rank == 0:
            _check(self.lib.tb_nccl_unique_id(uid), "tb_nccl_unique_id")
        obj = [bytes(uid.raw)]
        dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
        self._h = ctypes.c_void_p()
        _check(self.lib.tb_nccl_comm_init(ctypes.byref(self._h), ctypes.create_string_buffer(obj[0], 128),
                                          self.P, self.rank), "tb_nccl_comm_init")

    @property
    def handle(self) -> int:
        return self._h.value

    def close(self):
        if self._h is not None and self._h.value:
            _check(self.lib.tb_nccl_comm_destroy(self._h), "tb_nccl_comm_destroy")
        self._h = None
