"""CPU checks of the C-ABI boundary: the library loads and exports every
symbol include/tb_capi.h declares; host-side validation maps to ValueError."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "tb_capi.h")
LIB = os.path.join(ROOT, "paper_2512_16093_b200", "libtb200.so")


def declared_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char \*)\s*(tb_\w+)\s*\(", src, re.M)))


def test_header_declares_entry_points():
    names = declared_symbols()
    for must in ("tb_quantize_blockwise", "tb_w8a8_gemm", "tb_pool_block_means", "tb_kmean",
                 "tb_pool_quant_tokens", "tb_topk_blocks", "tb_sla_attention", "tb_last_error"):
        assert must in names


def test_library_exports_every_declared_symbol():
    if not os.path.exists(LIB):
        pytest.skip("libtb200.so not built (run __graft_entry__.build())")
    lib = ctypes.CDLL(LIB)
    missing = [n for n in declared_symbols() if not hasattr(lib, n)]
    assert not missing, missing


def test_python_binding_covers_header():
    from paper_2512_16093_b200 import _lib
    assert set(declared_symbols()) <= set(_lib.exported_symbols())


def test_host_validation_without_device():
    """Argument errors are caught host-side before any launch (TB_EINVAL -> ValueError)."""
    if not os.path.exists(LIB):
        pytest.skip("libtb200.so not built")
    from paper_2512_16093_b200 import _lib
    lib = _lib.load()
    rc = lib.tb_quantize_blockwise(None, 0, 4, 4, 0, None, None, None, None)
    assert rc == _lib.TB_EINVAL
    assert b"block" in lib.tb_last_error()
    rc = lib.tb_topk_blocks(None, None, 1, 1, 4, 8, 5, None, None, None, None)
    assert rc == _lib.TB_EINVAL
    with pytest.raises(ValueError):
        _lib.check(rc, "tb_topk_blocks")
    a = _lib.SlaArgs()
    a.H, a.L, a.d, a.q_block, a.kv_block, a.count = 1, 16, 8, 64, 64, 1
    assert lib.tb_sla_attention(ctypes.byref(a), None) == _lib.TB_EINVAL
    assert b"exceed" in lib.tb_last_error()


def test_sla_args_layout_matches_header():
    """ctypes mirror has the same field order/count as the C struct."""
    from paper_2512_16093_b200 import _lib
    src = open(HEADER).read()
    body = src[src.index("typedef struct tb_sla_args"):src.index("} tb_sla_args;")]
    body = re.sub(r"/\*.*?\*/", "", body, flags=re.S)
    fields = re.findall(r"\*?\s*(\w+)\s*[,;]", body.split("{", 1)[1])
    assert [f[0] for f in _lib.SlaArgs._fields_] == fields


def test_host_stage_copy_and_bf16_rounding():
    """tb_host_stage (host staging of numpy inputs): bit copies, and f32 -> bf16
    identical to torch's round-to-nearest-even cast incl. ties, inf, subnormals;
    NaN stays NaN.  Host-only entry point (no device needed)."""
    import numpy as np
    import torch
    from paper_2512_16093_b200 import _lib
    lib = _lib.load()
    rng = np.random.default_rng(0)
    for n in (0, 1, 17, 1000003, (1 << 18) * 3 + 5):
        x = (rng.standard_normal(n) * 3).astype(np.float32)
        if n > 20:
            x[:8] = [np.nan, np.inf, -np.inf, 0.0, -0.0, 1e-40, -1e-45, 3.4e38]
            x[9] = np.float32(1.00390625)                      # exact bf16 tie
            x[10] = np.float32(1.01171875)                     # tie, odd
        y = np.empty(n, dtype=np.uint16)
        assert lib.tb_host_stage(y.ctypes.data, x.ctypes.data, n, _lib.TB_F32, _lib.TB_BF16, 0) == 0
        ref = torch.from_numpy(x).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
        nan = np.isnan(x)
        assert np.array_equal(y[~nan], ref[~nan])
        assert np.all((y[nan] & 0x7F80) == 0x7F80) and np.all((y[nan] & 0x7F) != 0)
        z = np.empty_like(x)
        assert lib.tb_host_stage(z.ctypes.data, x.ctypes.data, n, _lib.TB_F32, _lib.TB_F32, 0) == 0
        assert np.array_equal(z.view(np.uint32), x.view(np.uint32))
    i8 = rng.integers(-128, 128, 12345, dtype=np.int8)
    o8 = np.empty_like(i8)
    assert lib.tb_host_stage(o8.ctypes.data, i8.ctypes.data, i8.size, _lib.TB_I8, _lib.TB_I8, 0) == 0
    assert np.array_equal(o8, i8)
    assert lib.tb_host_stage(o8.ctypes.data, i8.ctypes.data, i8.size, _lib.TB_I8, _lib.TB_F32, 0) == _lib.TB_EINVAL


def test_host_stage_bf16_exact_detects_and_narrows():
    """tb_host_stage_bf16_exact: bf16-valued f32 arrays (NaN / inf / -0.0 /
    subnormal bf16 values included) come back as their bf16 bit patterns with
    rc 1; one value with a nonzero low half anywhere (any span, any thread,
    head / tail / aligned body) gives rc 0."""
    import numpy as np
    import torch
    from paper_2512_16093_b200 import _lib
    lib = _lib.load()
    rng = np.random.default_rng(1)
    for n in (0, 1, 31, 1000003, (1 << 18) * 5 + 7):
        x = torch.from_numpy(rng.standard_normal(n).astype(np.float32)).to(torch.bfloat16).float().numpy()
        if n > 20:
            x[:6] = [np.nan, np.inf, -np.inf, -0.0, 9.18355e-41, 1.0]
            x[:6] = torch.from_numpy(x[:6]).to(torch.bfloat16).float().numpy()
        y = np.empty(n, dtype=np.uint16)
        assert lib.tb_host_stage_bf16_exact(y.ctypes.data, x.ctypes.data, n, 0) == 1
        assert np.array_equal(y, (x.view(np.uint32) >> 16).astype(np.uint16))
        for pos in sorted({0, n // 3, n - 1}) if n else []:
            z = x.copy()
            z.view(np.uint32)[pos] |= 1
            assert lib.tb_host_stage_bf16_exact(y.ctypes.data, z.ctypes.data, n, 0) == 0, (n, pos)


def test_sla_workspace_bytes_host_only():
    """tb_sla_workspace_bytes (SURVEY §8 b4 tb_workspace_bytes): sizes of every
    intermediate tb_sla_forward carves out of the caller's workspace, computed
    on the host (no device); bad ratios map to TB_EINVAL."""
    from paper_2512_16093_b200 import _lib
    lib = _lib.load()
    H, L, d = 40, 75600, 128
    nkv, nq = -(-L // 64), -(-L // 128)
    count = -(-int(0.1 * nkv * 10) // 10)
    n = lib.tb_sla_workspace_bytes(H, L, d, 128, 64, 0.1, 1.0, _lib.TB_BF16)
    # at least the codes, kv_part and KV_sel (the big ones)
    assert n >= 2 * H * L * d + H * nkv * 130 * d * 2 + H * nq * 130 * d * 2
    assert n < 4 * H * L * d + 2 * (H * nkv * 130 * d * 2) + (1 << 30)
    assert n % 256 == 0
    assert lib.tb_sla_workspace_bytes(H, L, d, 128, 64, 0.1, 1.0, _lib.TB_F32) > n     # + bf16 copies of k, v
    assert lib.tb_sla_workspace_bytes(H, L, d, 128, 64, 0.1, 0.0, _lib.TB_BF16) < n    # no linear branch
    assert lib.tb_sla_workspace_bytes(H, L, d, 64, 64, 0.1, 1.0, _lib.TB_BF16) > 0
    assert lib.tb_sla_workspace_bytes(H, L, d, 128, 64, 0.0, 1.0, _lib.TB_BF16) == _lib.TB_EINVAL
    assert lib.tb_sla_workspace_bytes(H, L, d, 128, 64, 1.5, 1.0, _lib.TB_BF16) == _lib.TB_EINVAL
    assert count == 119
