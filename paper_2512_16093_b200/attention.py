"""Drop-in for ``turbobench.attention`` (/root/reference/pkg/src/turbobench/attention.py).

Same names, dataclasses, argument meaning and errors as the reference; the
work runs in the sm_100a kernels of ``libtb200.so`` (via ``ops``).  numpy
inputs are uploaded to the current CUDA device and results come back as
numpy float32 (the reference's return type); torch CUDA tensors stay on the
device end to end.  ``sla_attention`` resolves ``select_topk_blocks`` and
the branch helpers through module globals, as the reference does
(attention.py:405-412), so monkeypatch-based fault injection keeps working.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import ops
from .blockquant import _F32_EXACT_BLOCK

__all__ = [
    "AttnInputs", "QuantAttnConfig", "SLAConfig", "BlockMask", "FlopReport",
    "reference_attention", "smooth_keys", "quantized_attention", "pool_block_means",
    "select_topk_blocks", "linear_attention", "sla_attention", "attention_flop_report",
    "instrumented_sparse_macs", "error_metrics",
]


def _device():
    return torch.device("cuda", torch.cuda.current_device())


def _is_torch(x) -> bool:
    return isinstance(x, torch.Tensor)


def _dev(x, dtype=torch.float32) -> torch.Tensor:
    """numpy / torch -> contiguous CUDA tensor (f32 unless bf16 given)."""
    if _is_torch(x):
        t = x if x.is_cuda else x.to(_device())
        if t.dtype not in (torch.float32, torch.bfloat16):
            t = t.float()
        return t.contiguous()
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).to(_device(), non_blocking=False)


def _ret(t: torch.Tensor, as_numpy: bool):
    return t.float().cpu().numpy() if as_numpy else t


@dataclass
class AttnInputs:
    """Query/key/value arrays of shape [heads, seq, head_dim] plus logit scale (attention.py:38-71)."""

    q: object
    k: object
    v: object
    scale: float | None = None

    def __post_init__(self):
        if not _is_torch(self.q):
            self.q = np.asarray(self.q, dtype=np.float32)
            self.k = np.asarray(self.k, dtype=np.float32)
            self.v = np.asarray(self.v, dtype=np.float32)
        if not (tuple(self.q.shape) == tuple(self.k.shape) == tuple(self.v.shape)) or self.q.ndim != 3:
            raise ValueError(
                f"q/k/v must share shape [heads, seq, head_dim], got "
                f"{tuple(self.q.shape)}, {tuple(self.k.shape)}, {tuple(self.v.shape)}")
        if self.q.shape[1] < 1 or self.q.shape[2] < 1:
            raise ValueError(f"seq and head_dim must be >= 1, got {tuple(self.q.shape)}")
        if self.scale is None:
            self.scale = 1.0 / math.sqrt(self.q.shape[2])

    @property
    def heads(self) -> int:
        return self.q.shape[0]

    @property
    def seq(self) -> int:
        return self.q.shape[1]

    @property
    def head_dim(self) -> int:
        return self.q.shape[2]

    @property
    def numpy_io(self) -> bool:
        return not _is_torch(self.q)


@dataclass
class QuantAttnConfig:
    token_block: int = 64
    smooth_k: bool = True

    def __post_init__(self):
        if self.token_block < 1:
            raise ValueError("token_block must be >= 1")


@dataclass
class SLAConfig:
    q_block: int = 64
    kv_block: int = 64
    topk_ratio: float = 0.1
    linear_mix: float = 1.0
    quantized_sparse_branch: bool = True

    def __post_init__(self):
        if not (0.0 < self.topk_ratio <= 1.0):
            raise ValueError(f"topk_ratio must be in (0, 1], got {self.topk_ratio}")
        if self.q_block < 1 or self.kv_block < 1:
            raise ValueError("block sizes must be >= 1")
        if self.linear_mix < 0:
            raise ValueError("linear_mix must be >= 0")


@dataclass
class BlockMask:
    """Selected kv-block indices per (head, query block), sorted ascending (attention.py:101-132)."""

    q_block: int
    kv_block: int
    num_kv_blocks: int
    indices: np.ndarray  # int64, [heads, num_q_blocks, count]

    @property
    def count(self) -> int:
        return self.indices.shape[2]

    def coverage(self) -> np.ndarray:
        h, nq, _ = self.indices.shape
        cov = np.zeros((h, nq, self.num_kv_blocks), dtype=bool)
        if self.count:
            np.put_along_axis(cov, np.asarray(self.indices), True, axis=-1)
        return cov

    def complement(self) -> "BlockMask":
        cov = self.coverage()
        m = self.num_kv_blocks - self.count
        idx = np.argsort(cov, axis=-1, kind="stable")[..., :m]
        return BlockMask(self.q_block, self.kv_block, self.num_kv_blocks, idx.astype(np.int64))


@dataclass
class FlopReport:
    dense_flops: int
    sparse_softmax_flops: int | None = None
    linear_branch_flops: int | None = None
    selection_overhead_flops: int | None = None
    dense_to_sparse_ratio: float | None = None

    def to_dict(self) -> dict:
        d = {"dense_flops": self.dense_flops}
        for key in ("sparse_softmax_flops", "linear_branch_flops",
                    "selection_overhead_flops", "dense_to_sparse_ratio"):
            val = getattr(self, key)
            if val is not None:
                d[key] = val
        return d


# ------------------------------------------------------------------ dense

def reference_attention(inputs: AttnInputs, return_probs: bool = False):
    """attention.py:161-176 -- dense f32 softmax attention (cuBLAS f32 GEMMs on device)."""
    q, k, v = _dev(inputs.q).float(), _dev(inputs.k).float(), _dev(inputs.v).float()
    logits = torch.bmm(q, k.transpose(1, 2)) * np.float32(inputs.scale)
    e = torch.exp(logits - logits.amax(dim=-1, keepdim=True))
    den = e.sum(dim=-1, keepdim=True)
    out = torch.bmm(e, v) / den
    if return_probs:
        return _ret(out, inputs.numpy_io), _ret(e / den, inputs.numpy_io)
    return _ret(out, inputs.numpy_io)


def smooth_keys(k):
    """attention.py:179-188 -> (k_centered, k_mean); k_mean is the bit-exact sequential mean."""
    numpy_io = not _is_torch(k)
    kd = _dev(k)
    km = ops.kmean(kd)
    kc = kd.float() - km[:, None, :]
    return _ret(kc, numpy_io), _ret(km, numpy_io)


def _quantize_token_blocks(x, block: int):
    """attention.py:201-220 -> (codes int8, scales f32), bit-exact."""
    numpy_io = not _is_torch(x)
    codes, scales, _ = ops.pool_quant_tokens(_dev(x), block, None, pool=False)
    if numpy_io:
        return codes.cpu().numpy(), scales.cpu().numpy()
    return codes, scales


def _exact_int_matmul_batched(a, b_t):
    """attention.py:223-227."""
    if a.shape[-1] <= _F32_EXACT_BLOCK:
        return np.matmul(np.asarray(a, np.float32), np.asarray(b_t, np.float32))
    return np.matmul(np.asarray(a, np.int64), np.asarray(b_t, np.int64)).astype(np.float32)


def pool_block_means(x, block: int):
    """attention.py:256-266, bit-exact (numpy reduceat order)."""
    if block < 1:
        raise ValueError("block must be >= 1")
    numpy_io = not _is_torch(x)
    return _ret(ops.pool_block_means(_dev(x), block), numpy_io)


def select_topk_blocks(qp, kp, cfg: SLAConfig) -> BlockMask:
    """attention.py:269-284, bit-exact indices (ties -> lower index)."""
    qpd, kpd = _dev(qp).float(), _dev(kp).float()
    num_kv = kpd.shape[1]
    count = math.ceil(cfg.topk_ratio * num_kv)
    idx, _, _ = ops.topk_blocks(qpd, kpd, count, want_comp=False)
    return BlockMask(q_block=cfg.q_block, kv_block=cfg.kv_block, num_kv_blocks=num_kv,
                     indices=idx.cpu().numpy().astype(np.int64))


def _feature_map(x):
    """attention.py:287-290."""
    if _is_torch(x):
        return torch.where(x >= 0, x + 1.0, torch.exp(torch.clamp(x, max=0.0)))
    return np.where(x >= 0.0, x + np.float32(1.0), np.exp(np.minimum(x, np.float32(0.0)))).astype(np.float32)


def _comp_from_mask(mask: BlockMask, heads: int) -> torch.Tensor:
    cov = torch.zeros((heads, mask.indices.shape[1], mask.num_kv_blocks), dtype=torch.uint8, device=_device())
    if mask.count:
        cov.scatter_(2, torch.from_numpy(np.asarray(mask.indices, np.int64)).to(_device()), 1)
    return cov


def linear_attention(inputs: AttnInputs, mask_complement: BlockMask | None = None):
    """attention.py:293-335 -> (numerator [h,s,d], denominator [h,s]) in f32."""
    q, k, v = _dev(inputs.q), _dev(inputs.k), _dev(inputs.v)
    h, s, d = q.shape
    if mask_complement is None:
        pack = ops.linear_branch(q, k, v, None, s, s, fast=False)
    else:
        nkv = -(-s // mask_complement.kv_block)
        if nkv != mask_complement.num_kv_blocks:
            raise ValueError("mask block count does not match the sequence")
        if mask_complement.count == 0:
            z = torch.zeros((h, s, d), device=q.device)
            return _ret(z, inputs.numpy_io), _ret(z[..., 0], inputs.numpy_io)
        comp = _comp_from_mask(mask_complement, h)
        pack = ops.linear_branch(q, k, v, comp, mask_complement.q_block, mask_complement.kv_block, fast=False)
    num, den = pack[:, :s, :d], pack[:, :s, d]
    return _ret(num.contiguous(), inputs.numpy_io), _ret(den.contiguous(), inputs.numpy_io)


def _gather_positions(sel_blocks, seq: int, block: int) -> np.ndarray:
    """attention.py:338-344."""
    parts = [np.arange(int(b) * block, min(int(b) * block + block, seq)) for b in sel_blocks]
    return np.concatenate(parts) if parts else np.empty(0, dtype=np.int64)


def _sparse_branch(inputs: AttnInputs, mask: BlockMask, cfg: SLAConfig):
    """attention.py:347-389 -> (num, den, row_max) with num/den carrying exp(-row_max)."""
    q, k, v = _dev(inputs.q), _dev(inputs.k), _dev(inputs.v)
    h, s, d = q.shape
    idx = torch.from_numpy(np.ascontiguousarray(mask.indices, np.int32)).to(q.device)
    count = idx.shape[2]
    kw = {}
    if cfg.quantized_sparse_branch:
        qc, qs, _ = ops.pool_quant_tokens(q, cfg.q_block, None, pool=False)
        km = ops.kmean(k)
        kc, ks, _ = ops.pool_quant_tokens(k, cfg.kv_block, km, pool=False)
        kw = dict(q_codes=ops.ptr(qc), k_codes=ops.ptr(kc), q_scales=ops.ptr(qs), k_scales=ops.ptr(ks),
                  k_mean=ops.ptr(km))
    out = torch.empty((h, s, d), device=q.device)
    row_max = torch.empty((h, s), device=q.device)
    den = torch.empty((h, s), device=q.device)
    # both kernels report (num/den, den, row_max) against the true row max (the
    # tensor-core one in its exact-max instantiation)
    kw.setdefault("vt", None)
    kw.update(ops.attention_operands(q, v, idx, cfg.q_block, cfg.kv_block, cfg.quantized_sparse_branch))
    args = ops.sla_args(q=ops.ptr(q), k=ops.ptr(k), v=ops.ptr(v), dtype=ops.dtype_code(q), H=h, L=s, d=d,
                        q_block=cfg.q_block, kv_block=cfg.kv_block, count=count, scale=float(inputs.scale),
                        linear_mix=0.0, quantized=int(cfg.quantized_sparse_branch), idx=ops.ptr(idx),
                        l_pad=0, num_l=None, den_l=None, out=ops.ptr(out), out_dtype=0, row_max=ops.ptr(row_max),
                        den=ops.ptr(den), **kw)
    import ctypes
    from . import _lib
    _lib.check(_lib.load(True).tb_sla_attention(ctypes.byref(args), ops.stream_ptr()), "tb_sla_attention")
    num = out * den[..., None]
    return _ret(num, inputs.numpy_io), _ret(den, inputs.numpy_io), _ret(row_max, inputs.numpy_io)


def quantized_attention(inputs: AttnInputs, cfg: QuantAttnConfig | None = None):
    """attention.py:230-253: dense INT8 Sage attention (every kv block selected)."""
    cfg = cfg or QuantAttnConfig()
    q, k, v = _dev(inputs.q), _dev(inputs.k), _dev(inputs.v)
    h, s, d = q.shape
    tb = min(cfg.token_block, s)        # a block longer than the sequence is one block of s tokens
    nb = -(-s // tb)
    qc, qs, _ = ops.pool_quant_tokens(q, tb, None, pool=False)
    km = ops.kmean(k) if cfg.smooth_k else torch.zeros((h, d), device=q.device)
    kc, ks, _ = ops.pool_quant_tokens(k, tb, km if cfg.smooth_k else None, pool=False)
    idx = torch.arange(nb, dtype=torch.int32, device=q.device).expand(h, nb, nb).contiguous()
    out = torch.empty((h, s, d), device=q.device)
    kw = {"vt": None}
    kw.update(ops.attention_operands(q, v, idx, tb, tb, True))
    args = ops.sla_args(q=ops.ptr(q), k=ops.ptr(k), v=ops.ptr(v), dtype=ops.dtype_code(q), H=h, L=s, d=d,
                        q_block=tb, kv_block=tb, count=nb, scale=float(inputs.scale), linear_mix=0.0, quantized=1,
                        q_codes=ops.ptr(qc), k_codes=ops.ptr(kc), q_scales=ops.ptr(qs), k_scales=ops.ptr(ks),
                        k_mean=ops.ptr(km), idx=ops.ptr(idx), l_pad=0, num_l=None, den_l=None,
                        out=ops.ptr(out), out_dtype=0, row_max=None, den=None, **kw)
    import ctypes
    from . import _lib
    _lib.check(_lib.load(True).tb_sla_attention(ctypes.byref(args), ops.stream_ptr()), "tb_sla_attention")
    return _ret(out, inputs.numpy_io)


def sla_attention(inputs: AttnInputs, cfg: SLAConfig | None = None):
    """attention.py:392-421: top-k block-sparse (INT8) softmax + linear branch on the complement.

    The fast path runs the whole pipeline on device (ops.sla_attention).  If
    ``select_topk_blocks`` has been replaced at module level (fault
    injection, test_verify.py:35-48) the mask comes from that callable.
    """
    cfg = cfg or SLAConfig()
    s = inputs.seq
    if cfg.q_block > s or cfg.kv_block > s:
        raise ValueError(f"block sizes {cfg.q_block}/{cfg.kv_block} exceed seq {s}")
    if select_topk_blocks is not _ORIG_SELECT:
        return _sla_with_mask(inputs, cfg)
    if inputs.numpy_io and inputs.heads > 1 and inputs.q.nbytes >= _HOST_PIPELINE_BYTES:
        # numpy in / numpy out at scale: per-head-chunk pipeline (staging copy,
        # upload, attention, download overlapped); same kernels, same values
        # the result array is backed by page-locked memory (torch's caching host
        # allocator), so the device->host copy lands in it directly
        out = torch.empty(inputs.q.shape, dtype=torch.float32, pin_memory=True)
        ops.sla_attention_host(torch.from_numpy(np.ascontiguousarray(inputs.q, np.float32)),
                               torch.from_numpy(np.ascontiguousarray(inputs.k, np.float32)),
                               torch.from_numpy(np.ascontiguousarray(inputs.v, np.float32)),
                               cfg.q_block, cfg.kv_block, cfg.topk_ratio, cfg.linear_mix,
                               cfg.quantized_sparse_branch, float(inputs.scale), out=out,
                               out_dtype=torch.float32, chunk_heads=_HOST_CHUNK_HEADS)
        torch.cuda.current_stream().synchronize()
        return out.numpy()
    q, k, v = _dev(inputs.q), _dev(inputs.k), _dev(inputs.v)
    out = ops.sla_attention(q, k, v, cfg.q_block, cfg.kv_block, cfg.topk_ratio, cfg.linear_mix,
                            cfg.quantized_sparse_branch, float(inputs.scale))
    return _ret(out, inputs.numpy_io)


_HOST_PIPELINE_BYTES = 64 << 20
_HOST_CHUNK_HEADS = 4          # heads per upload / attention / download chunk (4: 73-78 ms vs 74-80 for 2 at cfg4, profiles/r02_dropin_e2e_staging.log)


def _sla_with_mask(inputs: AttnInputs, cfg: SLAConfig):
    """Reference composition with module-global helpers (attention.py:405-421)."""
    qp = pool_block_means(inputs.q, cfg.q_block)
    kp = pool_block_means(inputs.k, cfg.kv_block)
    mask = select_topk_blocks(qp, kp, cfg)
    num_s, den_s, row_max = _sparse_branch(inputs, mask, cfg)
    comp = mask.complement()
    to = (lambda a: _dev(a)) if inputs.numpy_io else (lambda a: a)
    num_s, den_s, row_max = to(num_s), to(den_s), to(row_max)
    if comp.count == 0 or cfg.linear_mix == 0.0:
        return _ret(num_s / den_s[..., None], inputs.numpy_io)
    num_l, den_l = linear_attention(inputs, comp)
    num_l, den_l = to(num_l), to(den_l)
    ref = torch.clamp(row_max, min=0.0)
    sparse_scale = torch.exp(row_max - ref)
    shrink = torch.exp(-ref) * float(cfg.linear_mix)
    num = num_s * sparse_scale[..., None] + shrink[..., None] * num_l
    den = den_s * sparse_scale + shrink * den_l
    return _ret(num / den[..., None], inputs.numpy_io)


def attention_flop_report(seq: int, head_dim: int, heads: int, cfg: SLAConfig | None = None) -> FlopReport:
    """attention.py:424-457 (analytic; the algorithmic-work definition used by bench.py)."""
    if seq < 1 or head_dim < 1 or heads < 1:
        raise ValueError("dimensions must be positive")
    dense = 4 * heads * seq * seq * head_dim
    if cfg is None:
        return FlopReport(dense_flops=dense)
    nq = -(-seq // cfg.q_block)
    nkv = -(-seq // cfg.kv_block)
    count = math.ceil(cfg.topk_ratio * nkv)
    covered = min(count * cfg.kv_block, seq)
    sparse = 4 * heads * seq * covered * head_dim
    return FlopReport(dense_flops=dense, sparse_softmax_flops=sparse,
                      linear_branch_flops=4 * heads * seq * head_dim * head_dim,
                      selection_overhead_flops=2 * heads * nq * nkv * head_dim,
                      dense_to_sparse_ratio=dense / sparse)


def instrumented_sparse_macs(inputs: AttnInputs, cfg: SLAConfig) -> dict:
    """attention.py:460-479: MACs the sparse branch performs, tallied from the device mask."""
    qp = pool_block_means(inputs.q, cfg.q_block)
    kp = pool_block_means(inputs.k, cfg.kv_block)
    mask = select_topk_blocks(qp, kp, cfg)
    s, d = inputs.seq, inputs.head_dim
    ext = np.minimum((np.arange(mask.num_kv_blocks) + 1) * cfg.kv_block, s) - np.arange(mask.num_kv_blocks) * cfg.kv_block
    keys = ext[mask.indices].sum(axis=-1)                       # [h, nq] covered key positions
    rows = np.minimum((np.arange(mask.indices.shape[1]) + 1) * cfg.q_block, s) - np.arange(mask.indices.shape[1]) * cfg.q_block
    qk = int((keys * rows[None, :]).sum()) * d
    dense = 2 * inputs.heads * s * s * d
    return {"qk_macs": qk, "pv_macs": qk, "total_macs": 2 * qk, "dense_macs": dense}


def error_metrics(a, b) -> tuple[float, float]:
    """attention.py:482-495 (cosine, relative L2) in f64."""
    a = np.asarray(a.cpu() if _is_torch(a) else a, dtype=np.float32).ravel().astype(np.float64)
    b = np.asarray(b.cpu() if _is_torch(b) else b, dtype=np.float32).ravel().astype(np.float64)
    if a.shape != b.shape:
        raise ValueError(f"shape mismatch: {a.shape} vs {b.shape}")
    daa, dbb = float(np.dot(a, a)), float(np.dot(b, b))
    if daa == 0.0 or dbb == 0.0:
        raise ValueError("error metrics are undefined for zero-norm inputs")
    cosine = float(np.dot(a, b) / math.sqrt(daa * dbb))
    rel_l2 = float(np.linalg.norm(a - b) / math.sqrt(dbb))
    return cosine, rel_l2


def rel_l1(a, b) -> float:
    """North-star metric (not in the reference): sum|a-b| / sum|b|."""
    a = np.asarray(a.cpu() if _is_torch(a) else a, dtype=np.float64).ravel()
    b = np.asarray(b.cpu() if _is_torch(b) else b, dtype=np.float64).ravel()
    return float(np.abs(a - b).sum() / np.abs(b).sum())


_ORIG_SELECT = select_topk_blocks
