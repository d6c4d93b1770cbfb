"""Device-level operators: torch CUDA tensors in, torch CUDA tensors out.

Each function is a thin shim over one C-ABI entry point (include/tb_capi.h);
the CUDA kernels do the work.  The pipelines ``sla_attention`` and
``quantized_linear`` are also registered as ``torch.library`` custom ops
(``tb200::sla_attention``, ``tb200::quantized_linear``) so they compose with
torch code and CUDA graphs.  Nothing here runs on the CPU: inputs must live on
a CUDA device and the library must be built (no fallback).
"""
from __future__ import annotations

import math
import os
import time

import torch

from . import _lib
from ._lib import TB_BF16, TB_F32, TB_I8, call, dtype_code, ptr, stream_ptr


def cdiv(a: int, b: int) -> int:
    return -(-a // b)


def _dev_tensor(t: torch.Tensor, name: str) -> torch.Tensor:
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor")
    if t.dtype not in (torch.float32, torch.bfloat16):
        t = t.float()
    return t.contiguous()


def _empty(shape, dtype, like: torch.Tensor):
    return torch.empty(shape, dtype=dtype, device=like.device)


# ------------------------------------------------------------------- quant

def quantize_blockwise(x: torch.Tensor, block: int = 128, check_finite: bool = True):
    """blockquant.py:91-110 -> (codes int8 [r,c], scales f32 [ceil(r/b),ceil(c/b)])."""
    x = _dev_tensor(x, "x")
    if x.dim() != 2:
        raise ValueError(f"expected a matrix, got shape {tuple(x.shape)}")
    r, c = x.shape
    q = _empty((r, c), torch.int8, x)
    s = _empty((cdiv(r, block), cdiv(c, block)), torch.float32, x)
    flag = torch.zeros(1, dtype=torch.int32, device=x.device) if check_finite else None
    call("tb_quantize_blockwise", ptr(x), dtype_code(x), r, c, block, ptr(q), ptr(s), ptr(flag), stream_ptr())
    if check_finite and int(flag.item()) != 0:
        raise ValueError("input contains non-finite values")
    return q, s


def quantize_blockwise_planar(x: torch.Tensor):
    """quantize_blockwise (block 128) of the logical [L, P*128] matrix stored as
    P planes [L, 128] (a head-major attention output) -> (codes [L, P*128], scales)."""
    P, r, w = x.shape
    if w != 128:
        raise ValueError("planes must be 128 wide")
    c = P * 128
    q = _empty((r, c), torch.int8, x)
    s = _empty((cdiv(r, 128), P), torch.float32, x)
    call("tb_quantize_blockwise_planar", ptr(x.contiguous()), dtype_code(x), r, c, ptr(q), ptr(s), stream_ptr())
    return q, s


def dequantize_blockwise(q: torch.Tensor, scales: torch.Tensor, block: int):
    r, c = q.shape
    out = _empty((r, c), torch.float32, q)
    call("tb_dequantize_blockwise", ptr(q), ptr(scales.contiguous()), r, c, block, ptr(out), stream_ptr())
    return out


def transpose_codes(q: torch.Tensor) -> torch.Tensor:
    r, c = q.shape
    out = _empty((c, r), torch.int8, q)
    call("tb_transpose_codes", ptr(q.contiguous()), r, c, ptr(out), stream_ptr())
    return out


def w8a8_gemm(a_q, a_s, bt_q, b_s, block: int = 128, bias=None, out_dtype=torch.float32, exact: bool = True):
    """blockquant.py:132-161 (+ bias).  bt_q is the TRANSPOSED weight code matrix [N, K]."""
    M, K = a_q.shape
    N = bt_q.shape[0]
    if bt_q.shape[1] != K:
        raise ValueError(f"inner dims differ: {K} vs {bt_q.shape[1]}")
    out = _empty((M, N), out_dtype, a_q)
    fn = "tb_w8a8_gemm" if exact else "tb_w8a8_gemm_fast"
    call(fn, ptr(a_q.contiguous()), ptr(a_s.contiguous()), ptr(bt_q.contiguous()), ptr(b_s.contiguous()),
         ptr(None if bias is None else bias.float().contiguous()), M, N, K, block, ptr(out),
         TB_BF16 if out_dtype == torch.bfloat16 else TB_F32, stream_ptr())
    return out


def w8a8_gemm_ex(a_q, a_s, bt_q, b_s, block: int = 128, bias=None, out_dtype=torch.bfloat16, plane: int = 0,
                 act: int = 0):
    """Fast-mode W8A8 with epilogue options: plane > 0 stores the output as
    N/plane planes [M, plane] (qkv -> head-major [3, H, M, head_dim]); act=1
    applies GELU-tanh."""
    M, K = a_q.shape
    N = bt_q.shape[0]
    if bt_q.shape[1] != K:
        raise ValueError(f"inner dims differ: {K} vs {bt_q.shape[1]}")
    out = _empty((N // plane, M, plane) if plane else (M, N), out_dtype, a_q)
    call("tb_w8a8_gemm_fast_ex", ptr(a_q.contiguous()), ptr(a_s.contiguous()), ptr(bt_q.contiguous()),
         ptr(b_s.contiguous()), ptr(None if bias is None else bias.float().contiguous()), M, N, K, block, ptr(out),
         TB_BF16 if out_dtype == torch.bfloat16 else TB_F32, plane, act, stream_ptr())
    return out


def w8a8_gemm_qkv_peers(a_q, a_s, bt_q, b_s, peers, heads: int, row0: int, L: int, block: int = 128, bias=None):
    """Fused Ulysses forward exchange: the qkv projection of this rank's token
    rows [row0, row0 + M) stored straight into the head owners' buffers
    (``peers``: P device addresses of bf16 [3*H/P, L, 128] buffers, peer memory
    on a multi-GPU box)."""
    import ctypes
    M, K = a_q.shape
    N = bt_q.shape[0]
    if bt_q.shape[1] != K:
        raise ValueError(f"inner dims differ: {K} vs {bt_q.shape[1]}")
    arr = (ctypes.c_void_p * len(peers))(*[int(p) for p in peers])
    call("tb_w8a8_gemm_qkv_peers", ptr(a_q.contiguous()), ptr(a_s.contiguous()), ptr(bt_q.contiguous()),
         ptr(b_s.contiguous()), ptr(None if bias is None else bias.float().contiguous()), M, N, K, block,
         ctypes.cast(arr, ctypes.c_void_p), len(peers), heads, row0, L, stream_ptr())


def w8a8_gemm_quant(a_q, a_s, bt_q, b_s, block: int = 128, bias=None, act: int = 0):
    """Fast-mode W8A8 (+ GELU when act=1) whose result is block-quantized for the
    next projection -> (codes int8 [M, N], scales [ceil(M/128), N/128]); equal to
    quantize_blockwise(w8a8_gemm_ex(..., bf16, act=act)).  One kernel (the
    quantization in the GEMM epilogue) where the 2-SM kernel applies."""
    M, K = a_q.shape
    N = bt_q.shape[0]
    if bt_q.shape[1] != K:
        raise ValueError(f"inner dims differ: {K} vs {bt_q.shape[1]}")
    if not (block == 128 and K % 128 == 0 and N % 256 == 0 and M >= 256):
        h = w8a8_gemm_ex(a_q, a_s, bt_q, b_s, block, bias, torch.bfloat16, act=act)
        return quantize_blockwise(h, block, check_finite=False)
    q = _empty((M, N), torch.int8, a_q)
    sc = _empty((cdiv(M, 128), N // 128), torch.float32, a_q)
    call("tb_w8a8_gemm_quant", ptr(a_q.contiguous()), ptr(a_s.contiguous()), ptr(bt_q.contiguous()),
         ptr(b_s.contiguous()), ptr(None if bias is None else bias.float().contiguous()), M, N, K, block, act,
         ptr(q), ptr(sc), stream_ptr())
    return q, sc


def quantized_linear(x, bt_q, b_s, block: int = 128, bias=None, out_dtype=torch.float32, exact: bool = True,
                     check_finite: bool = False):
    """quantized_linear_forward (blockquant.py:164-182): activation quant + W8A8."""
    xq, xs = quantize_blockwise(x, block, check_finite=check_finite)
    return w8a8_gemm(xq, xs, bt_q, b_s, block, bias, out_dtype, exact)


# ------------------------------------------------------ SLA block importance

def pool_block_means(x: torch.Tensor, block: int) -> torch.Tensor:
    """attention.py:256-266 (numpy reduceat order)."""
    x = _dev_tensor(x, "x")
    H, L, d = x.shape
    out = _empty((H, cdiv(L, block), d), torch.float32, x)
    call("tb_pool_block_means", ptr(x), dtype_code(x), H, L, d, block, ptr(out), stream_ptr())
    return out


def kmean(k: torch.Tensor) -> torch.Tensor:
    """attention.py:187 (sequential chain over tokens)."""
    k = _dev_tensor(k, "k")
    H, L, d = k.shape
    out = _empty((H, d), torch.float32, k)
    call("tb_kmean", ptr(k), dtype_code(k), H, L, d, ptr(out), stream_ptr())
    return out


def quant_v_fp8(v: torch.Tensor):
    """V [H, L, d] -> (e4m3 codes uint8 [H, L, d], per-head scales f32 [H]) for the
    opt-in FP8 P/V path (rule in include/tb_capi.h)."""
    v = _dev_tensor(v, "v")
    H, L, d = v.shape
    codes = _empty((H, L, d), torch.uint8, v)
    scales = _empty((H,), torch.float32, v)
    ws = _empty((max(H, 1),), torch.int32, v)
    call("tb_quant_v_fp8", ptr(v), dtype_code(v), H, L, d, ptr(codes), ptr(scales), ptr(ws), stream_ptr())
    return codes, scales


def pool_quant_tokens(x: torch.Tensor, block: int, center: torch.Tensor | None = None, pool: bool = True):
    """attention.py:201-220 (+ fused pooling of raw x) -> (codes, scales, pooled|None)."""
    x = _dev_tensor(x, "x")
    H, L, d = x.shape
    nb = cdiv(L, block)
    codes = _empty((H, L, d), torch.int8, x)
    scales = _empty((H, nb), torch.float32, x)
    pooled = _empty((H, nb, d), torch.float32, x) if pool else None
    call("tb_pool_quant_tokens", ptr(x), dtype_code(x), ptr(center), H, L, d, block, ptr(codes), ptr(scales),
         ptr(pooled), stream_ptr())
    return codes, scales, pooled


def pool_quant_tokens_t(x: torch.Tensor, block: int, center: torch.Tensor | None = None):
    """pool_quant_tokens plus the pooled means transposed [H, d, ldt] (the
    top-k kernel's coalesced kp operand) -> (codes, scales, pooled, pooled_t)."""
    x = _dev_tensor(x, "x")
    H, L, d = x.shape
    nb = cdiv(L, block)
    ldt = -(-nb // 4) * 4
    codes = _empty((H, L, d), torch.int8, x)
    scales = _empty((H, nb), torch.float32, x)
    pooled = _empty((H, nb, d), torch.float32, x)
    pooled_t = _empty((H, d, ldt), torch.float32, x)
    call("tb_pool_quant_tokens_t", ptr(x), dtype_code(x), ptr(center), H, L, d, block, ptr(codes), ptr(scales),
         ptr(pooled), ptr(pooled_t), ldt, stream_ptr())
    return codes, scales, pooled, pooled_t


def pool_tokens_t(x: torch.Tensor, block: int):
    """pool_block_means (attention.py:256-266) of raw x, plus the transposed
    [H, d, ldt] copy for the coalesced top-k kernel -> (pooled, pooled_t)."""
    x = _dev_tensor(x, "x")
    H, L, d = x.shape
    nb = cdiv(L, block)
    ldt = -(-nb // 4) * 4
    pooled = _empty((H, nb, d), torch.float32, x)
    pooled_t = _empty((H, d, ldt), torch.float32, x)
    call("tb_pool_quant_tokens_t", ptr(x), dtype_code(x), None, H, L, d, block, None, None,
         ptr(pooled), ptr(pooled_t), ldt, stream_ptr())
    return pooled, pooled_t


def topk_count(ratio: float, nkv: int) -> int:
    """attention.py:279."""
    return math.ceil(ratio * nkv)


def topk_blocks(qp: torch.Tensor, kp: torch.Tensor, count: int, want_comp: bool = True,
                want_scores: bool = False):
    """attention.py:269-284 + 122-132 -> (idx int32 [H,nq,count], comp uint8|None, scores|None)."""
    qp, kp = qp.float().contiguous(), kp.float().contiguous()
    H, nq, d = qp.shape
    nkv = kp.shape[1]
    idx = _empty((H, nq, count), torch.int32, qp)
    comp = _empty((H, nq, nkv), torch.uint8, qp) if want_comp else None
    scores = _empty((H, nq, nkv), torch.float32, qp) if want_scores else None
    call("tb_topk_blocks", ptr(qp), ptr(kp), H, nq, nkv, d, count, ptr(idx), ptr(comp), ptr(scores), stream_ptr())
    return idx, comp, scores


def topk_blocks_cov(qp: torch.Tensor, kp: torch.Tensor, count: int, want_comp: bool = False,
                    kpt: torch.Tensor | None = None):
    """select_topk_blocks + the complement as the bf16 coverage matrix of the
    linear branch's GEMM -> (idx, comp uint8|None, cov bf16 [H, nq, nkv_pad]).
    kpt: kp transposed [H, d, ldk] (pool_quant_tokens_t) for the fast path."""
    qp, kp = qp.float().contiguous(), kp.float().contiguous()
    H, nq, d = qp.shape
    nkv = kp.shape[1]
    ld = -(-nkv // 8) * 8                            # TMA row pitch must be a multiple of 16 B
    idx = _empty((H, nq, count), torch.int32, qp)
    comp = _empty((H, nq, nkv), torch.uint8, qp) if want_comp else None
    cov = _empty((H, nq, ld), torch.bfloat16, qp)
    call("tb_topk_blocks_cov", ptr(qp), ptr(kp), ptr(kpt), 0 if kpt is None else kpt.shape[2], H, nq, nkv, d,
         count, ptr(idx), ptr(comp), ptr(cov), ld, stream_ptr())
    return idx, comp, cov


def pair_union(idx: torch.Tensor):
    """tb_pair_union: union of the top-k lists of q-block pairs (2t, 2t+1) for
    the q_block 64 tensor-core kernel -> (pair_idx int32 [H, ceil(nq/2),
    2*count], entries block | mask << 28; pair_cnt int32 [H, ceil(nq/2)])."""
    H, nq, count = idx.shape
    nt = cdiv(nq, 2)
    pidx = _empty((H, nt, 2 * count), torch.int32, idx)
    pcnt = _empty((H, nt), torch.int32, idx)
    call("tb_pair_union", ptr(idx), H, nq, count, ptr(pidx), ptr(pcnt), 2 * count, stream_ptr())
    return pidx, pcnt


def cast_bf16(x: torch.Tensor) -> torch.Tensor:
    """tb_cast_bf16: f32 -> bf16 (RN), same shape."""
    x = x.contiguous()
    y = torch.empty(x.shape, dtype=torch.bfloat16, device=x.device)
    call("tb_cast_bf16", ptr(x), x.numel(), ptr(y), stream_ptr())
    return y


def attention_operands(q: torch.Tensor, v: torch.Tensor, idx: torch.Tensor, q_block: int, kv_block: int,
                       quantized: bool) -> dict:
    """The extra tb_sla_args a direct tb_sla_attention call needs for the
    tensor-core kernel to serve it: the bf16 V copy when the inputs are f32,
    and the pair-union lists for q_block 64.  Returns sla_args keywords (vt,
    pair_*); an empty dict keeps the call on the CUDA-core kernel.  The
    pointers are taken last (ptr() keeps each tensor alive until the next C
    call returns, so no call may run between them and tb_sla_attention)."""
    H, L, d = q.shape
    count = idx.shape[2]
    if not tc_envelope(H, L, d, q_block, kv_block, count, quantized):
        return {}
    vt = cast_bf16(v) if q.dtype == torch.float32 else None
    pidx = pcnt = None
    if q_block == 64:
        pidx, pcnt = pair_union(idx)
    return dict(vt=ptr(vt), pair_idx=ptr(pidx), pair_cnt=ptr(pcnt), pair_ld=0 if pidx is None else pidx.shape[2])


def tc_envelope(H: int, L: int, d: int, q_block: int, kv_block: int, count: int, quantized: bool = True) -> bool:
    """Shapes the tcgen05 attention kernel serves (csrc/sla_tc.cu
    sla_tc_supported): head_dim 128, kv_block 64, q_block 128, or q_block 64
    (the reference default) with at most 2048 union blocks per 128-row tile."""
    nkv = cdiv(L, kv_block)
    return (quantized and d == 128 and kv_block == 64 and L >= 128 and 1 <= count <= 2048 and
            (q_block == 128 or (q_block == 64 and min(2 * count, nkv) <= 2048)))


def transpose_v(v: torch.Tensor, l_pad: int) -> torch.Tensor:
    v = _dev_tensor(v, "v")
    H, L, d = v.shape
    vt = _empty((H, d, l_pad), torch.bfloat16, v)
    call("tb_transpose_v", ptr(v), dtype_code(v), H, L, d, l_pad, ptr(vt), stream_ptr())
    return vt


def feature_map(x: torch.Tensor, l_pad: int, out_dtype=torch.float32) -> torch.Tensor:
    """phi (attention.py:287-290) into [H, l_pad, d]; padding rows are 0."""
    x = _dev_tensor(x, "x")
    H, L, d = x.shape
    out = _empty((H, l_pad, d), out_dtype, x)
    call("tb_feature_map", ptr(x), dtype_code(x), H, L, d, l_pad, ptr(out),
         TB_BF16 if out_dtype == torch.bfloat16 else TB_F32, stream_ptr())
    return out


def linear_operands(q, k, v, lq: int, lk: int, dx: int, dtype=torch.bfloat16, lvt: int = 0, linear: bool = True,
                    want_phiq: bool = True):
    """tb_linear_operands -> (phiq [H,lq,d], phik [H,lk,d], vext [H,lk,dx] = [v | 1 | 0], vt [H,d,lvt] | None)."""
    q, k, v = _dev_tensor(q, "q"), _dev_tensor(k, "k"), _dev_tensor(v, "v")
    H, L, d = q.shape
    phiq = _empty((H, lq, d), dtype, q) if (linear and want_phiq) else None
    phik = _empty((H, lk, d), dtype, q) if linear else None
    vext = _empty((H, lk, dx), dtype, q) if linear else None
    vt = _empty((H, d, lvt), torch.bfloat16, q) if lvt else None
    call("tb_linear_operands", ptr(q), ptr(k), ptr(v), dtype_code(q), H, L, d, lq, lk, dx, ptr(phiq), ptr(phik),
         ptr(vext), TB_BF16 if dtype == torch.bfloat16 else TB_F32, ptr(vt), lvt, stream_ptr())
    return phiq, phik, vext, vt


def linear_kv_dx(d: int) -> int:
    """Rows of a kv_part block: d numerator rows, the denominator row, and
    zero padding up to the smallest dx with dx*d a multiple of 256 (the
    coverage GEMM's N tile)."""
    dx = d + 1
    while (dx * d) % 256:
        dx += 1
    return dx


def linear_kv_part(k, v, kv_block: int, pool: bool = False, k_mean=None):
    """tb_linear_kv_part: per kv block [V_b | 1]^T phi(K_b) (attention.py:320-325)
    straight from bf16 k, v -> [H, nkv, dx, d] bf16 (one tcgen05 kernel).
    pool=True (tb_linear_kv_part_pool): also the raw K block means and their
    transposed copy from the same tiles -> (kv_part, kp, kpt), as pool_tokens_t.
    k_mean given (with pool=True; tb_linear_kv_part_codes): also the smoothed K
    codes and scales -> (kv_part, kp, kpt, kc, ks), as pool_quant_tokens(k, kv_block, k_mean)."""
    H, L, d = k.shape
    nkv = cdiv(L, kv_block)
    dx = linear_kv_dx(d)
    kv_part = torch.empty((H, nkv, dx, d), dtype=torch.bfloat16, device=k.device)
    if not pool:
        call("tb_linear_kv_part", ptr(k), ptr(v), H, L, d, kv_block, dx, ptr(kv_part), stream_ptr())
        return kv_part
    ldt = -(-nkv // 4) * 4
    kp = torch.empty((H, nkv, d), dtype=torch.float32, device=k.device)
    kpt = torch.empty((H, d, ldt), dtype=torch.float32, device=k.device)
    if k_mean is None:
        call("tb_linear_kv_part_pool", ptr(k), ptr(v), H, L, d, kv_block, dx, ptr(kv_part), ptr(kp), ptr(kpt), ldt,
             stream_ptr())
        return kv_part, kp, kpt
    kc = torch.empty((H, L, d), dtype=torch.int8, device=k.device)
    ks = torch.empty((H, nkv), dtype=torch.float32, device=k.device)
    call("tb_linear_kv_part_codes", ptr(k), ptr(v), H, L, d, kv_block, dx, ptr(kv_part), ptr(kp), ptr(kpt), ldt,
         ptr(k_mean), ptr(kc), ptr(ks), stream_ptr())
    return kv_part, kp, kpt, kc, ks


def linear_kv_sel(kv_part: torch.Tensor, cov: torch.Tensor, nkv: int):
    """Fused-epilogue form of the linear branch (attention.py:320-328).

    Returns kvsel [H, nq, dx, d] bf16: per q block n, rows 0..d-1 hold
    KV_sel[n]^T = sum over complement blocks b of V_b^T phi(K_b), row d holds
    sum phi(K_b); the attention kernel finishes the branch with one tcgen05
    MMA phi(Q_n) . KV_sel[n] in its epilogue (attention.py:329-334).  The
    coverage GEMM cov . kv_part is ours (tb_gemm_bf16_batched), bf16 operands
    with f32 accumulation.
    """
    H, _, dx, d = kv_part.shape
    nq = cov.shape[1]
    kvsel = gemm_bf16_batched(cov, kv_part.view(H, nkv, dx * d), K=nkv)         # [H, nq, dx*d]
    return kvsel.view(H, nq, dx, d)


def gemm_bf16_batched(a: torch.Tensor, b: torch.Tensor, K: int | None = None, out_dtype=torch.bfloat16):
    """tb_gemm_bf16_batched: C[h] = A[h][:, :K] . B[h][:K] (tcgen05, f32 accumulate)."""
    H, M, lda = a.shape
    Kb, N = b.shape[1], b.shape[2]
    K = Kb if K is None else K
    c = torch.empty((H, M, N), dtype=out_dtype, device=a.device)
    call("tb_gemm_bf16_batched", ptr(a), ptr(b), ptr(c), H, M, N, K, lda, N, N,
         TB_F32 if out_dtype == torch.float32 else TB_BF16, stream_ptr())
    return c


def linear_branch(q, k, v, comp: torch.Tensor | None, q_block: int, kv_block: int, fast: bool = False,
                  lvt: int = 0):
    """linear_attention over the complement mask (attention.py:293-335) on CUDA
    cores (tb_linear_branch_simt), for shapes outside the tensor-core envelope
    (which runs kv_part + the coverage GEMM + the attention kernel's fused
    MMA instead).

    comp: uint8 [H, nq, nkv] (1 = block in the complement) or None for the
    unmasked form.  Returns the packed f32 tensor [H, lq, dx] (columns
    0..d-1 = numerator, column d = denominator) with lq = nq*q_block (or L
    when comp is None).  ``fast`` / ``lvt`` are accepted for API stability
    (the CUDA-core path is f32 only and needs no V^T)."""
    q, k, v = _dev_tensor(q, "q"), _dev_tensor(k, "k"), _dev_tensor(v, "v")
    if k.dtype != q.dtype or v.dtype != q.dtype:
        k, v = k.to(q.dtype), v.to(q.dtype)
    H, L, d = q.shape
    dx = -(-(d + 1) // 16) * 16
    if comp is None:
        q_block = kv_block = L
        nq = nkv = 1
    else:
        nq, nkv = comp.shape[1], comp.shape[2]
        comp = comp.to(torch.uint8).contiguous()
    part = torch.empty((H, nkv, d, d + 1), dtype=torch.float32, device=q.device)
    sel = torch.empty((H, nq, d, d + 1), dtype=torch.float32, device=q.device)
    out = torch.empty((H, nq * q_block, dx), dtype=torch.float32, device=q.device)
    call("tb_linear_branch_simt", ptr(q), ptr(k), ptr(v), dtype_code(q), H, L, d, ptr(comp), nq, nkv, q_block,
         kv_block, ptr(part), ptr(sel), ptr(out), dx, stream_ptr())
    if lvt:
        return out, None
    return out


_SIDE = {}
# kernel the last ops.sla_attention call ran ("tcgen05" / "cuda_core"; tests)
LAST_SLA_PATH = None


def _km_event(side: torch.cuda.Stream) -> torch.cuda.Event:
    """An event recorded on the side stream right after k_mean was enqueued
    (sla_attention records it before the kv_part launch)."""
    return _KM_EVENT[torch.cuda.current_device()]


_KM_EVENT = {}


def _side_stream() -> torch.cuda.Stream:
    dev = torch.cuda.current_device()
    s = _SIDE.get(dev)
    if s is None:
        s = _SIDE[dev] = torch.cuda.Stream(device=dev)
    return s


def sla_args(**kw) -> _lib.SlaArgs:
    a = _lib.SlaArgs()
    for key, val in kw.items():
        setattr(a, key, val)
    return a


def sla_attention(q, k, v, q_block: int = 64, kv_block: int = 64, topk_ratio: float = 0.1,
                  linear_mix: float = 1.0, quantized: bool = True, scale: float | None = None,
                  out_dtype=torch.float32, linear_fast: bool | None = None, return_parts: bool = False,
                  pv_fp8: bool = False, peer_out: dict | None = None):
    """sla_attention (attention.py:392-421) on device tensors [H, L, d].

    pv_fp8: opt-in FP8 P/V -- V quantized to e4m3 with
    per-head scales (quant_v_fp8) and the PV product as kind::f8f6f4 on e4m3
    P; tensor-core envelope and bf16 inputs only.  Off by default: FP8 P/V
    misses rel-L1 <= 1e-2 when the sparse branch dominates (Appendix A.6).

    peer_out (out_dtype int8 only): the fused Ulysses return path -- dict with
    ``codes`` / ``scales``: int64 device tensors [P] of the owners' buffer
    addresses (peer memory), ``rows`` (token-shard rows, multiple of 128),
    ``head0`` (global index of this shard's first head), ``heads`` (global H).
    The epilogue stores every tile in its token owner's buffers; returns None."""
    q, k, v = _dev_tensor(q, "q"), _dev_tensor(k, "k"), _dev_tensor(v, "v")
    if not (q.shape == k.shape == v.shape) or q.dim() != 3:
        raise ValueError(f"q/k/v must share shape [heads, seq, head_dim], got "
                         f"{tuple(q.shape)}, {tuple(k.shape)}, {tuple(v.shape)}")
    H, L, d = q.shape
    if q_block > L or kv_block > L:
        raise ValueError(f"block sizes {q_block}/{kv_block} exceed seq {L}")
    scale = 1.0 / math.sqrt(d) if scale is None else float(scale)
    nq, nkv = cdiv(L, q_block), cdiv(L, kv_block)
    count = topk_count(topk_ratio, nkv)
    parts = {}
    lin = count < nkv and linear_mix != 0.0
    tc = tc_envelope(H, L, d, q_block, kv_block, count, quantized)
    if k.dtype != q.dtype:
        k = k.to(q.dtype)
    # f32 q / k with a bf16 V is accepted on the tensor-core path, which reads
    # V only as bf16 (PV operand, linear-branch kv_part): the host pipeline
    # ships V already rounded (sla_attention_host), same values as the cast below
    if v.dtype != q.dtype and not (tc and q.dtype == torch.float32 and v.dtype == torch.bfloat16):
        v = v.to(q.dtype)
    l_pad = nkv * 64
    main = torch.cuda.current_stream()
    # bf16 tensor-core path with the linear branch: the pool pass also emits
    # kp transposed for the coalesced top-k kernel, which writes the bf16
    # coverage matrix for the branch's GEMM
    fast_lin = lin and tc and quantized and q.dtype == torch.bfloat16
    kpt = None
    # the tensor-core path reads V (and the linear-branch kernel K and V) as bf16
    kb = k if k.dtype == torch.bfloat16 else cast_bf16(k)
    vb = v if v.dtype == torch.bfloat16 else cast_bf16(v)
    vt = None if q.dtype == torch.bfloat16 else vb
    # Side stream: k_mean (a latency-bound sequential chain) and the linear
    # branch's per-block operand kv_part (HBM-bound, needs only k and v) run
    # under the Q / K passes and the (issue-bound) top-k selection.
    side = _side_stream()
    side.wait_stream(main)
    kv_part = lin_pack = lin_kv = cov = None
    v8 = v8s = None
    if pv_fp8 and not (tc and q.dtype == torch.bfloat16):
        raise ValueError("FP8 P/V needs bf16 inputs on the tensor-core path (d=128, q_block 128 or 64, kv_block=64)")
    if fast_lin:
        # Three streams.  The top-k selection needs only the pooled raw K
        # (attention.py:404-406), so the main stream runs Q pass -> K pooling ->
        # top-k -> coverage GEMM without waiting for k_mean; k_mean (a
        # sequential chain) and the K codes that need it run on the side
        # stream, kv_part (HBM-bound, needs only k and v) on a third from t=0.
        # _KV_POOL: kv_part also pools the raw K blocks from the tiles it holds
        # (no separate K pooling pass) and top-k waits for it after the Q pass
        # _KV_CODES (opt-in): kv_part also writes the smoothed K codes from those
        # tiles (no separate K pass), so it starts once k_mean is done
        third = _aux_stream("kvpart")
        third.wait_stream(main)
        codes_in_kv = _KV_POOL and _KV_CODES
        if codes_in_kv:
            with torch.cuda.stream(side):
                km = kmean(k)
            third.wait_stream(side)
        with torch.cuda.stream(third):
            if codes_in_kv:
                kv_part, kp, kpt, kc, ks = linear_kv_part(kb, vb, kv_block, pool=True, k_mean=km)
                km.record_stream(third)
            elif _KV_POOL:
                kv_part, kp, kpt = linear_kv_part(kb, vb, kv_block, pool=True)
            else:
                kv_part = linear_kv_part(kb, vb, kv_block)
            ev_kv = torch.cuda.Event()
            ev_kv.record(third)
            if pv_fp8:                                  # V codes only need v
                v8, v8s = quant_v_fp8(v)
        if not codes_in_kv:
            with torch.cuda.stream(side):
                km = kmean(k)
                kc, ks, _ = pool_quant_tokens(k, kv_block, km, pool=False)
        qc, qs, qp = pool_quant_tokens(q, q_block, None, pool=True)
        if _KV_POOL:
            main.wait_event(ev_kv)
            for t in (kp, kpt):
                t.record_stream(main)
        else:
            kp, kpt = pool_tokens_t(k, kv_block)
        idx, comp, cov = topk_blocks_cov(qp, kp, count, want_comp=return_parts, kpt=kpt)
        main.wait_stream(third)
        kv_part.record_stream(main)
        if pv_fp8:
            v8.record_stream(main)
            v8s.record_stream(main)
        lin_kv = linear_kv_sel(kv_part, cov, nkv)
        main.wait_stream(side)
        for t in (km, kc, ks):
            t.record_stream(main)
    else:
        # Side stream: k_mean (a latency-bound sequential chain) and, for the
        # tensor-core path, the linear branch's per-block operand kv_part
        with torch.cuda.stream(side):
            km = kmean(k) if quantized else None
            ev = _KM_EVENT.setdefault(torch.cuda.current_device(), torch.cuda.Event())
            ev.record(side)
            if lin and tc:
                kv_part = linear_kv_part(kb, vb, kv_block)
        if quantized:
            qc, qs, qp = pool_quant_tokens(q, q_block, None, pool=True)
            main.wait_stream(side) if not (lin and tc) else main.wait_event(_km_event(side))
            km.record_stream(main)
            kc, ks, kp = pool_quant_tokens(k, kv_block, km, pool=True)
        else:
            qc = qs = kc = ks = None
            qp, kp = pool_block_means(q, q_block), pool_block_means(k, kv_block)
        if lin and tc:
            idx, comp, cov = topk_blocks_cov(qp, kp, count, want_comp=return_parts, kpt=None)
            main.wait_stream(side)
            kv_part.record_stream(main)
            lin_kv = linear_kv_sel(kv_part, cov, nkv)
        else:
            idx, comp, _ = topk_blocks(qp, kp, count, want_comp=lin or return_parts)
            if lin:
                fast = (H * L * d >= (1 << 22)) if linear_fast is None else linear_fast
                lin_pack = linear_branch(q, k, v, comp, q_block, kv_block, fast=fast)
    if pv_fp8 and v8 is None:
        v8, v8s = quant_v_fp8(v)
    pidx = pcnt = None
    if tc and q_block == 64:
        pidx, pcnt = pair_union(idx)
    q8 = out_dtype == torch.int8
    if q8 and not (tc and not return_parts):
        raise ValueError("int8 output (quantized out-projection operand) needs the tensor-core path")
    if peer_out is not None and not q8:
        raise ValueError("peer output needs out_dtype int8")
    # int8: codes [L, H*d] + scales [nq, H] of the bf16-rounded output (the
    # out-projection's block-quantized A operand, written by the epilogue)
    if peer_out is not None:
        out = out_scales = None
    else:
        out = (torch.empty((L, H * d), dtype=torch.int8, device=q.device) if q8
               else torch.empty((H, L, d), dtype=out_dtype, device=q.device))
        out_scales = torch.empty((cdiv(L, 128), H), dtype=torch.float32, device=q.device) if q8 else None
    row_max = torch.empty((H, L), dtype=torch.float32, device=q.device) if return_parts else None
    den = torch.empty((H, L), dtype=torch.float32, device=q.device) if return_parts else None
    args = sla_args(q=ptr(q), k=ptr(k), v=ptr(v), dtype=dtype_code(q), H=H, L=L, d=d, q_block=q_block,
                    kv_block=kv_block, count=count, scale=scale, linear_mix=float(linear_mix),
                    quantized=int(bool(quantized)), q_codes=ptr(qc), k_codes=ptr(kc), q_scales=ptr(qs),
                    k_scales=ptr(ks), k_mean=ptr(km), idx=ptr(idx), vt=ptr(vt), l_pad=l_pad,
                    num_l=ptr(lin_pack), den_l=None,
                    lin_ld=0 if lin_pack is None else lin_pack.shape[2],
                    lin_hs=0 if lin_pack is None else lin_pack.shape[1] * lin_pack.shape[2],
                    lin_kv=ptr(lin_kv), lin_dx=0 if lin_kv is None else lin_kv.shape[2], out=ptr(out),
                    out_dtype=TB_I8 if q8 else (TB_BF16 if out_dtype == torch.bfloat16 else TB_F32),
                    row_max=ptr(row_max), den=ptr(den), out_scales=ptr(out_scales),
                    v_fp8=ptr(v8), v_scales=ptr(v8s), pair_idx=ptr(pidx), pair_cnt=ptr(pcnt),
                    pair_ld=0 if pidx is None else pidx.shape[2])
    if peer_out is not None:
        args.out_peers, args.scale_peers = ptr(peer_out["codes"]), ptr(peer_out["scales"])
        args.peer_rows, args.head0, args.out_heads = int(peer_out["rows"]), int(peer_out["head0"]), int(peer_out["heads"])
    lib = _lib.load(require_device=True)
    global LAST_SLA_PATH
    LAST_SLA_PATH = "tcgen05" if lib.tb_sla_path(__import__("ctypes").byref(args)) == 1 else "cuda_core"
    _lib.check(lib.tb_sla_attention(__import__("ctypes").byref(args), stream_ptr()), "tb_sla_attention")
    if return_parts:
        parts = dict(qp=qp, kp=kp, idx=idx, comp=comp, q_codes=qc, q_scales=qs, k_codes=kc, k_scales=ks,
                     k_mean=km, lin_pack=lin_pack, lin_kv=lin_kv, row_max=row_max, den=den, count=count,
                     v_fp8=v8, v_scales=v8s)
        return out, parts
    if peer_out is not None:
        return None
    return (out, out_scales) if q8 else out


def sla_forward(q, k, v, q_block: int = 64, kv_block: int = 64, topk_ratio: float = 0.1, linear_mix: float = 1.0,
                scale: float | None = None, out_dtype=torch.float32):
    """The single-call C-ABI pipeline (tb_sla_forward: every prep pass and the
    fused kernel, intermediates in one workspace from tb_sla_workspace_bytes)
    on device tensors [H, L, d] -- what a non-Python host binds.  Same kernels
    and values as sla_attention on the tensor-core envelope."""
    q, k, v = _dev_tensor(q, "q"), _dev_tensor(k, "k"), _dev_tensor(v, "v")
    if not (q.shape == k.shape == v.shape) or q.dim() != 3:
        raise ValueError("q/k/v must share shape [heads, seq, head_dim]")
    if k.dtype != q.dtype:
        k = k.to(q.dtype)
    if v.dtype != q.dtype:
        v = v.to(q.dtype)
    H, L, d = q.shape
    scale = 1.0 / math.sqrt(d) if scale is None else float(scale)
    lib = _lib.load(require_device=True)
    nbytes = lib.tb_sla_workspace_bytes(H, L, d, q_block, kv_block, float(topk_ratio), float(linear_mix),
                                        dtype_code(q))
    if nbytes < 0:
        _lib.check(int(nbytes), "tb_sla_workspace_bytes")
    ws = torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=q.device)
    out = torch.empty((H, L, d), dtype=out_dtype, device=q.device)
    call("tb_sla_forward", ptr(q), ptr(k), ptr(v), dtype_code(q), H, L, d, q_block, kv_block, float(topk_ratio),
         float(linear_mix), scale, ptr(ws), int(nbytes), ptr(out), TB_BF16 if out_dtype == torch.bfloat16 else TB_F32,
         stream_ptr())
    return out


_AUX = {}

# bf16 tensor-core path: the raw K pool comes from kv_part's tiles (True) or
# from a separate pooling pass on the caller's stream (False; tools A/B)
_KV_POOL = True
_KV_CODES = False   # measured slower: kv_part would wait for k_mean


def _aux_stream(name: str) -> torch.cuda.Stream:
    key = (torch.cuda.current_device(), name)
    s = _AUX.get(key)
    if s is None:
        s = _AUX[key] = torch.cuda.Stream()
    return s


_HOST_CODES = {torch.float32: TB_F32, torch.bfloat16: TB_BF16, torch.int8: TB_I8}


def host_stage(dst: torch.Tensor, src: torch.Tensor) -> torch.Tensor:
    """dst.copy_(src) for contiguous HOST tensors on the library's pool of
    host threads with non-temporal stores (tb_host_stage); f32 -> bf16 rounds
    to nearest even like torch's cast.  Other layouts / dtypes: torch's copy."""
    sc, dc = _HOST_CODES.get(src.dtype), _HOST_CODES.get(dst.dtype)
    if (src.is_cuda or dst.is_cuda or sc is None or dc is None or dst.shape != src.shape
            or not (src.is_contiguous() and dst.is_contiguous()) or not (sc == dc or (sc, dc) == (TB_F32, TB_BF16))):
        return dst.copy_(src)
    call("tb_host_stage", dst.data_ptr(), src.data_ptr(), src.numel(), sc, dc, 0)
    return dst


# tools: set to a dict to accumulate sla_attention_host's host wall time per
# phase (stage / wait_upload / enqueue / wait_d2h), seconds
HOST_PROFILE: dict | None = None

# bytes the last sla_attention_host call moved across PCIe (and how many head
# chunks took the lossless bf16 upload), for the e2e report
LAST_HOST_TRANSFER: dict = {}


def sla_attention_host(q, k, v, q_block: int = 64, kv_block: int = 64, topk_ratio: float = 0.1,
                       linear_mix: float = 1.0, quantized: bool = True, scale: float | None = None,
                       out: torch.Tensor | None = None, out_dtype=torch.bfloat16, chunk_heads: int = 4):
    """sla_attention on HOST tensors [H, L, d]: every hot-path quantity is
    per head (attention.py:370), so the heads are processed in chunks and the
    host->device copy of chunk i+1, the attention of chunk i and the
    device->host copy of chunk i-1 run on three streams at once.

    Pinned inputs / output are copied directly.  Pageable ones (numpy-backed,
    what the drop-in receives) are staged through two pinned buffers per
    tensor: the host copies chunk i+1 into its staging buffer while the GPU
    works on chunk i, and copies chunk i-1's result out of the output staging
    buffer once its device->host copy is done.  Returns ``out``."""
    if q.is_cuda or k.is_cuda or v.is_cuda:
        raise ValueError("sla_attention_host takes host tensors; use sla_attention for device tensors")
    if not (q.shape == k.shape == v.shape) or q.dim() != 3:
        raise ValueError(f"q/k/v must share shape [heads, seq, head_dim], got "
                         f"{tuple(q.shape)}, {tuple(k.shape)}, {tuple(v.shape)}")
    H, L, d = q.shape
    pinned_in = q.is_pinned() and k.is_pinned() and v.is_pinned()
    if out is None:
        out = torch.empty((H, L, d), dtype=out_dtype, pin_memory=True)
    pinned_out = out.is_pinned()
    dev = torch.device("cuda", torch.cuda.current_device())
    compute = torch.cuda.current_stream()
    h2d, d2h = _aux_stream("h2d"), _aux_stream("d2h")
    h2d.wait_stream(compute)
    d2h.wait_stream(compute)
    ch = max(1, min(chunk_heads, H))
    # f32 inputs on the tensor-core path: V crosses PCIe already rounded to bf16
    # (the kernels read V only as bf16), half its bytes
    nkv = cdiv(L, kv_block)
    v_half = (q.dtype == torch.float32 and not pinned_in and
              tc_envelope(ch, L, d, q_block, kv_block, topk_count(topk_ratio, nkv), quantized))
    dts = (q.dtype, k.dtype, torch.bfloat16 if v_half else v.dtype)
    # bf16-valued f32 q / k (a bf16 model's activations handed over as f32
    # arrays) cross PCIe as their exact bf16 bit patterns, checked per chunk
    # while staging (tb_host_stage_bf16_exact); the bf16 kernels widen them
    # back exactly, so the result is the f32 path's.  Anything else ships f32.
    narrow = v_half and k.dtype == torch.float32 and q.is_contiguous() and k.is_contiguous()
    bufs = [[torch.empty((ch, L, d), dtype=dt, device=dev) for dt in dts] for _ in range(2)]
    stage_in = None if pinned_in else \
        [[torch.empty((ch, L, d), dtype=dt, pin_memory=True) for dt in dts] for _ in range(2)]
    stage_out = None if pinned_out else [torch.empty((ch, L, d), dtype=out.dtype, pin_memory=True) for _ in range(2)]
    ev_in = [torch.cuda.Event() for _ in range(2)]
    ev_done = [torch.cuda.Event() for _ in range(2)]
    ev_out = [torch.cuda.Event() for _ in range(2)]
    pending = None                                       # (buffer, h0, h1) of a staged output not yet copied out
    moved = LAST_HOST_TRANSFER
    # chunk boundaries: a one-head chunk first and last (the pipeline's fill --
    # staging + upload of chunk 0 -- and drain -- attention + download of the
    # last chunk -- are not overlapped with anything), ch heads in between
    bounds = _chunk_bounds(H, ch)
    moved.update(h2d_bytes=0, d2h_bytes=0, narrow_chunks=0, chunks=len(bounds))

    prof = HOST_PROFILE                                  # optional per-phase host wall times (tools)
    tick = time.perf_counter if prof is not None else None

    def mark(key, t0):
        if prof is not None:
            prof[key] = prof.get(key, 0.0) + tick() - t0

    def finish(p):
        b_, a_, z_ = p
        t0 = tick() if tick else 0.0
        ev_out[b_].synchronize()
        mark("wait_d2h", t0)
        out[a_:z_].copy_(stage_out[b_][:z_ - a_])

    def stage(i):
        """chunk i's (sources, device destinations); pageable inputs are first
        staged into page-locked buffer i % 2 (bf16 bit patterns when exact)"""
        h0, h1 = bounds[i]
        n, b = h1 - h0, i % 2
        srcs = (q[h0:h1], k[h0:h1], v[h0:h1])
        dsts = tuple(t[:n] for t in bufs[b])
        if stage_in is None:
            return srcs, dsts
        torch.cuda.set_device(dev)                       # the worker thread's device
        t0 = tick() if tick else 0.0
        if i >= 2:
            ev_in[b].synchronize()                       # chunk i-2's upload has left staging buffer b
        mark("wait_upload", t0)
        t0 = tick() if tick else 0.0
        sq, sk = _bf16_view(stage_in[b][0], n), _bf16_view(stage_in[b][1], n)
        if narrow and host_stage_bf16_exact(sq, srcs[0]) and host_stage_bf16_exact(sk, srcs[1]):
            host_stage(stage_in[b][2][:n], srcs[2])
            srcs = (sq, sk, stage_in[b][2][:n])
            dsts = (_bf16_view(bufs[b][0], n), _bf16_view(bufs[b][1], n), bufs[b][2][:n])
        else:
            for st_, src in zip(stage_in[b], srcs):
                host_stage(st_[:n], src)
            srcs = tuple(st_[:n] for st_ in stage_in[b])
        mark("stage", t0)
        return srcs, dsts

    nch = len(bounds)
    # staging of chunk i+1 (host threads, GIL released in the native call) runs
    # on a worker while this thread enqueues chunk i's upload / attention / download
    worker = _stage_worker() if stage_in is not None and nch > 1 else None
    staged = stage(0)
    for i in range(nch):
        h0, h1 = bounds[i]
        n, b = h1 - h0, i % 2
        nxt = worker.submit(stage, i + 1) if worker is not None and i + 1 < nch else None
        srcs, dsts = staged
        t0 = tick() if tick else 0.0
        if i >= 2:
            h2d.wait_event(ev_done[b])                  # chunk i-2 has consumed device buffer b
        moved["h2d_bytes"] += sum(t.numel() * t.element_size() for t in srcs)
        moved["narrow_chunks"] += int(dsts[0].dtype == torch.bfloat16 and q.dtype == torch.float32)
        with torch.cuda.stream(h2d):
            for dst, src in zip(dsts, srcs):
                dst.copy_(src, non_blocking=True)
            ev_in[b].record(h2d)
        compute.wait_event(ev_in[b])
        o = sla_attention(dsts[0], dsts[1], dsts[2], q_block, kv_block, topk_ratio,
                          linear_mix, quantized, scale, out_dtype=out.dtype)
        ev_done[b].record(compute)
        d2h.wait_event(ev_done[b])
        with torch.cuda.stream(d2h):
            (out[h0:h1] if stage_out is None else stage_out[b][:n]).copy_(o, non_blocking=True)
            ev_out[b].record(d2h)
        o.record_stream(d2h)
        moved["d2h_bytes"] += o.numel() * o.element_size()
        mark("enqueue", t0)
        if pending is not None:
            finish(pending)                              # chunk i-1: its result is (being) copied out
        pending = (b, h0, h1) if stage_out is not None else None
        if i + 1 < nch:
            t0 = tick() if tick else 0.0
            staged = nxt.result() if nxt is not None else stage(i + 1)
            mark("join_stage", t0)
    if pending is not None:
        finish(pending)
    for bb in bufs:
        for t in bb:
            t.record_stream(compute)
            t.record_stream(h2d)
    compute.wait_stream(d2h)                            # the caller's stream covers the output copy
    return out


_HOST_EDGE_CHUNKS = True        # single-head first / last chunks (tools A/B)


def _chunk_bounds(H: int, ch: int) -> list[tuple[int, int]]:
    """Head ranges of sla_attention_host's chunks: [0, 1), then ch heads at a
    time, the last chunk again a single head (H > ch + 1)."""
    if H <= ch + 1 or ch <= 1 or not _HOST_EDGE_CHUNKS:
        return [(h, min(H, h + ch)) for h in range(0, H, ch)]
    out, h = [(0, 1)], 1
    while h < H - 1:
        out.append((h, min(H - 1, h + ch)))
        h = out[-1][1]
    out.append((H - 1, H))
    return out


_WORKER = {}


def _stage_worker():
    """One background thread per process for sla_attention_host's staging."""
    import concurrent.futures
    pid = os.getpid()
    w = _WORKER.get(pid)
    if w is None:
        w = _WORKER[pid] = concurrent.futures.ThreadPoolExecutor(max_workers=1, thread_name_prefix="tb-stage")
    return w


def _bf16_view(t: torch.Tensor, n: int) -> torch.Tensor:
    """The first n heads' worth of a [ch, L, d] f32 buffer's bytes as a bf16 [n, L, d] tensor."""
    return t.view(-1).view(torch.bfloat16)[: n * t.shape[1] * t.shape[2]].view(n, t.shape[1], t.shape[2])


def host_stage_bf16_exact(dst: torch.Tensor, src: torch.Tensor) -> bool:
    """Stage contiguous host f32 ``src`` into host bf16 ``dst`` when every value
    is exactly representable in bf16 (tb_host_stage_bf16_exact): True and dst
    holds the same values, or False (dst unspecified) -- the lossless narrow
    upload encoding of bf16-valued f32 inputs."""
    if (src.is_cuda or dst.is_cuda or src.dtype != torch.float32 or dst.dtype != torch.bfloat16
            or dst.shape != src.shape or not (src.is_contiguous() and dst.is_contiguous())):
        raise ValueError("host_stage_bf16_exact takes contiguous host f32 -> bf16 tensors of one shape")
    rc = _lib.load().tb_host_stage_bf16_exact(dst.data_ptr(), src.data_ptr(), src.numel(), 0)
    if rc < 0:
        _lib.check(int(rc), "tb_host_stage_bf16_exact")
    return rc == 1


# ------------------------------------------------------------------ DiT rows

def rmsnorm(x, gain, eps=1e-6):
    x = x.float().contiguous()
    out = torch.empty_like(x)
    r, c = x.shape
    call("tb_rmsnorm", ptr(x), ptr(gain.float().contiguous()), r, c, float(eps), ptr(out), stream_ptr())
    return out


def layernorm(x, gain, offset, eps=1e-6):
    x = x.float().contiguous()
    out = torch.empty_like(x)
    r, c = x.shape
    call("tb_layernorm", ptr(x), ptr(gain.float().contiguous()), ptr(offset.float().contiguous()), r, c,
         float(eps), ptr(out), stream_ptr())
    return out


def add_norm(x, y=None, emb=None, alpha: float = 0.0, gain=None, offset=None, layer_norm: bool = False,
             eps: float = 1e-6, sum_out=None, write_sum: bool = True):
    """s = x (+ y) (+ alpha*emb) -> (s f32 | None, norm(s) bf16) in one pass (DiT glue)."""
    rows, cols = x.shape
    if write_sum and sum_out is None:
        sum_out = torch.empty_like(x)
    norm = torch.empty((rows, cols), dtype=torch.bfloat16, device=x.device)
    call("tb_add_norm", ptr(x), ptr(y), ptr(emb), float(alpha), ptr(gain), ptr(offset), rows, cols, float(eps),
         int(layer_norm), ptr(sum_out if write_sum else None), ptr(norm), stream_ptr())
    return (sum_out if write_sum else None), norm


def add_norm_quant(x, y=None, emb=None, alpha: float = 0.0, gain=None, offset=None, layer_norm: bool = False,
                   eps: float = 1e-6, sum_out=None, write_sum: bool = True):
    """add_norm fused with quantize_blockwise(., 128) of the bf16 norm output
    (tb_add_norm_quant): -> (s f32 | None, codes int8 [rows, cols], scales
    [ceil(rows/128), cols/128]), bit-identical to add_norm + quantize_blockwise
    with one HBM pass.  cols % 128 == 0 and cols <= 6144."""
    rows, cols = x.shape
    if write_sum and sum_out is None:
        sum_out = torch.empty_like(x)
    q = torch.empty((rows, cols), dtype=torch.int8, device=x.device)
    sc = torch.empty((cdiv(rows, 128), cols // 128), dtype=torch.float32, device=x.device)
    call("tb_add_norm_quant", ptr(x), ptr(y), ptr(emb), float(alpha), ptr(gain), ptr(offset), rows, cols,
         float(eps), int(layer_norm), ptr(sum_out if write_sum else None), ptr(q), ptr(sc), stream_ptr())
    return (sum_out if write_sum else None), q, sc


def add_norm_quant_ok(cols: int) -> bool:
    return cols % 128 == 0 and 128 <= cols <= 6144


def axpy_rn(acc: torch.Tensor, x: torch.Tensor, c: float) -> torch.Tensor:
    """acc += fl(c * x) in place (f32, two RN roundings; merge.py:68)."""
    assert acc.dtype == torch.float32 and x.dtype == torch.float32 and acc.is_contiguous()
    call("tb_axpy_rn", ptr(acc), ptr(x.contiguous()), float(c), acc.numel(), stream_ptr())
    return acc


def gelu(x):
    x = x.float().contiguous()
    out = torch.empty_like(x)
    call("tb_gelu", ptr(x), x.numel(), ptr(out), stream_ptr())
    return out


# --------------------------------------------------- torch.library registration

@torch.library.custom_op("tb200::sla_attention", mutates_args=())
def _sla_attention_op(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, q_block: int, kv_block: int,
                      topk_ratio: float, linear_mix: float, quantized: bool) -> torch.Tensor:
    return sla_attention(q, k, v, q_block, kv_block, topk_ratio, linear_mix, quantized)


@_sla_attention_op.register_fake
def _(q, k, v, q_block, kv_block, topk_ratio, linear_mix, quantized):
    return torch.empty(q.shape, dtype=torch.float32, device=q.device)


@torch.library.custom_op("tb200::quantized_linear", mutates_args=())
def _quantized_linear_op(x: torch.Tensor, bt_q: torch.Tensor, b_s: torch.Tensor, block: int,
                         bias: torch.Tensor | None, exact: bool) -> torch.Tensor:
    return quantized_linear(x, bt_q, b_s, block, bias, torch.float32, exact)


@_quantized_linear_op.register_fake
def _(x, bt_q, b_s, block, bias, exact):
    return torch.empty((x.shape[0], bt_q.shape[0]), dtype=torch.float32, device=x.device)
