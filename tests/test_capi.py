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
