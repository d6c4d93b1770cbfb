"""ctypes binding of the C ABI (include/tb_capi.h) -> libtb200.so.

The library is built in-tree (``make -C paper_2512_16093_b200/csrc``) and
loaded from the package directory.  There is no fallback: if the library or
a CUDA device is missing, every op raises.
"""
from __future__ import annotations

import ctypes
import threading
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# TB200_LIB selects an alternative in-tree build (e.g. the phase-trace variant)
LIB_PATH = os.environ.get("TB200_LIB") or os.path.join(_HERE, "libtb200.so")

TB_OK, TB_EINVAL, TB_ECUDA, TB_EUNSUPPORTED = 0, -1, -2, -3
TB_F32, TB_BF16, TB_I8 = 0, 1, 2

_P = ctypes.c_void_p
_I = ctypes.c_int64
_i = ctypes.c_int
_f = ctypes.c_float

# exported symbol -> argtypes (restype int unless listed in _RESTYPES)
SIGNATURES = {
    "tb_last_error": [],
    "tb_device_ok": [],
    "tb_build_info": [],
    "tb_quantize_blockwise": [_P, _i, _I, _I, _I, _P, _P, _P, _P],
    "tb_quantize_blockwise_planar": [_P, _i, _I, _I, _P, _P, _P],
    "tb_dequantize_blockwise": [_P, _P, _I, _I, _I, _P, _P],
    "tb_transpose_codes": [_P, _I, _I, _P, _P],
    "tb_w8a8_gemm": [_P, _P, _P, _P, _P, _I, _I, _I, _I, _P, _i, _P],
    "tb_w8a8_gemm_fast": [_P, _P, _P, _P, _P, _I, _I, _I, _I, _P, _i, _P],
    "tb_w8a8_gemm_quant": [_P, _P, _P, _P, _P, _I, _I, _I, _I, _i, _P, _P, _P],
    "tb_w8a8_gemm_qkv_peers": [_P, _P, _P, _P, _P, _I, _I, _I, _I, _P, _I, _I, _I, _I, _P],
    "tb_w8a8_gemm_fast_ex": [_P, _P, _P, _P, _P, _I, _I, _I, _I, _P, _i, _I, _i, _P],
    "tb_quantized_linear": [_P, _i, _P, _P, _P, _I, _I, _I, _I, _P, _P, _P, _i, _P],
    "tb_pool_block_means": [_P, _i, _I, _I, _I, _I, _P, _P],
    "tb_kmean": [_P, _i, _I, _I, _I, _P, _P],
    "tb_pool_quant_tokens": [_P, _i, _P, _I, _I, _I, _I, _P, _P, _P, _P],
    "tb_topk_blocks": [_P, _P, _I, _I, _I, _I, _I, _P, _P, _P, _P],
    "tb_topk_blocks_cov": [_P, _P, _P, _I, _I, _I, _I, _I, _I, _P, _P, _P, _I, _P],
    "tb_pool_quant_tokens_t": [_P, _i, _P, _I, _I, _I, _I, _P, _P, _P, _P, _I, _P],
    "tb_sla_attention": [_P, _P],
    "tb_pair_union": [_P, _I, _I, _I, _P, _P, _I, _P],
    "tb_cast_bf16": [_P, _I, _P, _P],
    "tb_host_stage": [_P, _P, _I, _i, _i, _I],
    "tb_host_threads": [],
    "tb_host_stage_bf16_exact": [_P, _P, _I, _I],
    "tb_timestamp": [_P, _P],
    "tb_sla_workspace_bytes": [_I, _I, _I, _I, _I, ctypes.c_double, _f, _i],
    "tb_sla_forward": [_P, _P, _P, _i, _I, _I, _I, _I, _I, ctypes.c_double, _f, _f, _P, _I, _P, _i, _P],
    "tb_sla_path": [_P],
    "tb_ulysses_shard": [_I, _I, _I],
    "tb_ulysses_workspace_bytes": [_I, _I, _I, _I, _I, _I],
    "tb_ulysses_seq_to_heads": [_P, _I, _I, _I, _I, _I, _I, _I, _P, _P, _P, _P, _i, _P],
    "tb_ulysses_heads_to_seq": [_P, _I, _I, _I, _I, _I, _I, _I, _P, _P, _P, _P, _i, _P],
    "tb_nccl_unique_id": [_P],
    "tb_nccl_comm_init": [_P, _P, _I, _I],
    "tb_nccl_comm_destroy": [_P],
    "tb_linear_branch_simt": [_P, _P, _P, _i, _I, _I, _I, _P, _I, _I, _I, _I, _P, _P, _P, _I, _P],
    "tb_transpose_v": [_P, _i, _I, _I, _I, _I, _P, _P],
    "tb_quant_v_fp8": [_P, _i, _I, _I, _I, _P, _P, _P, _P],
    "tb_peer_alloc": [_I, _P],
    "tb_peer_free": [_P],
    "tb_peer_export": [_P, _P],
    "tb_peer_import": [_P, _P],
    "tb_peer_close": [_P],
    "tb_peer_barrier": [_P, _I, _I, ctypes.c_uint32, _P],
    "tb_feature_map": [_P, _i, _I, _I, _I, _I, _P, _i, _P],
    "tb_linear_operands": [_P, _P, _P, _i, _I, _I, _I, _I, _I, _I, _P, _P, _P, _i, _P, _I, _P],
    "tb_gemm_bf16_batched": [_P, _P, _P, _I, _I, _I, _I, _I, _I, _I, _i, _P],
    "tb_linear_kv_part": [_P, _P, _I, _I, _I, _I, _I, _P, _P],
    "tb_linear_kv_part_pool": [_P, _P, _I, _I, _I, _I, _I, _P, _P, _P, _I, _P],
    "tb_linear_kv_part_codes": [_P, _P, _I, _I, _I, _I, _I, _P, _P, _P, _I, _P, _P, _P, _P],
    "tb_rmsnorm": [_P, _P, _I, _I, _f, _P, _P],
    "tb_axpy_rn": [_P, _P, _f, _I, _P],
    "tb_add_norm": [_P, _P, _P, _f, _P, _P, _I, _I, _f, _i, _P, _P, _P],
    "tb_add_norm_quant": [_P, _P, _P, _f, _P, _P, _I, _I, _f, _i, _P, _P, _P, _P],
    "tb_layernorm": [_P, _P, _P, _I, _I, _f, _P, _P],
    "tb_gelu": [_P, _I, _P, _P],
}
_RESTYPES = {"tb_last_error": ctypes.c_char_p, "tb_build_info": ctypes.c_char_p,
             "tb_ulysses_shard": ctypes.c_int64, "tb_host_threads": ctypes.c_int64, "tb_sla_workspace_bytes": ctypes.c_int64, "tb_ulysses_workspace_bytes": ctypes.c_int64}


class SlaArgs(ctypes.Structure):
    """Mirror of ``tb_sla_args`` (include/tb_capi.h)."""
    _fields_ = [
        ("q", _P), ("k", _P), ("v", _P),
        ("dtype", _i),
        ("H", _I), ("L", _I), ("d", _I), ("q_block", _I), ("kv_block", _I), ("count", _I),
        ("scale", _f), ("linear_mix", _f),
        ("quantized", _i),
        ("q_codes", _P), ("k_codes", _P),
        ("q_scales", _P), ("k_scales", _P),
        ("k_mean", _P),
        ("idx", _P),
        ("vt", _P),
        ("l_pad", _I),
        ("num_l", _P), ("den_l", _P),
        ("lin_ld", _I), ("lin_hs", _I),
        ("lin_kv", _P), ("lin_dx", _I),
        ("out", _P),
        ("out_dtype", _i),
        ("row_max", _P), ("den", _P),
        ("out_scales", _P),
        ("v_fp8", _P), ("v_scales", _P),
        ("out_peers", _P), ("scale_peers", _P),
        ("peer_rows", _I), ("head0", _I), ("out_heads", _I),
        ("pair_idx", _P), ("pair_cnt", _P), ("pair_ld", _I),
    ]


_lib = None


def load(require_device: bool = False):
    """Load libtb200.so (raises if absent)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built: run `make -C {os.path.join(_HERE, 'csrc')}` "
                              "(or __graft_entry__.build()); there is no CPU fallback")
        lib = ctypes.CDLL(LIB_PATH)
        for name, args in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = _RESTYPES.get(name, ctypes.c_int)
        _lib = lib
    if require_device:
        if not torch.cuda.is_available():
            raise RuntimeError("paper_2512_16093_b200 needs a CUDA device (B200, sm_100a); no CPU fallback")
        if _lib.tb_device_ok() != 1:
            raise RuntimeError("libtb200.so is built for sm_100a only; the visible device is not a B200")
    return _lib


def exported_symbols():
    return list(SIGNATURES)


def check(rc: int, what: str):
    _release()
    if rc == TB_OK:
        return
    msg = load().tb_last_error().decode(errors="replace")
    if rc == TB_EINVAL:
        raise ValueError(msg or what)
    raise RuntimeError(f"{what}: {msg} (status {rc})")


def call(name: str, *args):
    lib = load(require_device=True)
    check(getattr(lib, name)(*args), name)


_KEEP = threading.local()


def ptr(t: torch.Tensor | None):
    """Raw device address of ``t`` for a C-ABI argument list.  The tensor is
    kept alive until the next ``call`` / ``check`` returns: call sites pass
    temporaries (``ptr(x.contiguous())``), and a temporary freed before its
    kernel is enqueued could be handed by the caching allocator to the next
    temporary in the same argument list and overwritten before the kernel
    reads it.  Once the kernel is enqueued, stream order makes the free safe."""
    if t is None:
        return None
    keep = getattr(_KEEP, "items", None)
    if keep is None:
        keep = _KEEP.items = []
    keep.append(t)
    return ctypes.c_void_p(t.data_ptr())


def _release():
    keep = getattr(_KEEP, "items", None)
    if keep:
        keep.clear()


def stream_ptr():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def dtype_code(t: torch.Tensor) -> int:
    if t.dtype == torch.float32:
        return TB_F32
    if t.dtype == torch.bfloat16:
        return TB_BF16
    raise ValueError(f"unsupported dtype {t.dtype} (need float32 or bfloat16)")
