"""TBT1 tensor files and manifests: the reference's format tests
(tests/test_tensor_store.py in the reference) restated against this package, the
reference-written fixtures in tests/golden/tbt (make_golden_tbt.py), and the
streamed pinned -> HBM loader on the GPU."""
import os
import struct

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

from paper_2512_16093_b200 import tensor_store as ts

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "tbt")


def test_shape1_file_is_18_bytes(tmp_path):
    ts.write_tensor(np.zeros(1, np.float32), tmp_path / "s.tbt")
    assert (tmp_path / "s.tbt").stat().st_size == 18


def test_header_bytes(tmp_path):
    ts.write_tensor(np.array([[1, 2, 3], [4, 5, 6]], np.int8), tmp_path / "i.tbt")
    assert (tmp_path / "i.tbt").read_bytes() == b"TBT1" + bytes([1, 2]) + struct.pack("<QQ", 2, 3) + bytes(
        [1, 2, 3, 4, 5, 6])


@pytest.mark.parametrize("dtype", [np.float32, np.int8])
@pytest.mark.parametrize("shape", [(1,), (7,), (3, 4), (2, 3, 4), (2, 2, 2, 3)])
def test_roundtrip_bits(tmp_path, dtype, shape):
    rng = np.random.default_rng(0)
    a = rng.standard_normal(shape).astype(dtype) if dtype == np.float32 else rng.integers(
        -128, 128, shape).astype(np.int8)
    ts.write_tensor(a, tmp_path / "t.tbt")
    b = ts.read_tensor(tmp_path / "t.tbt")
    assert b.dtype == a.dtype and b.shape == a.shape
    assert np.array_equal(b.view(np.uint8), a.view(np.uint8))


@given(st.lists(st.integers(1, 5), min_size=1, max_size=4), st.integers(0, 2**32))
@settings(max_examples=25, deadline=None)
def test_roundtrip_property(tmp_path_factory, dims, seed):
    a = np.random.default_rng(seed).standard_normal(dims).astype(np.float32)
    p = tmp_path_factory.mktemp("rt") / "t.tbt"
    ts.write_tensor(a, p)
    assert np.array_equal(ts.read_tensor(p), a)
    assert p.stat().st_size == 6 + 8 * a.ndim + 4 * a.size


@pytest.mark.parametrize("raw,err", [
    (b"XXXX" + bytes(20), ts.BadMagicError),
    (b"TB", ts.BadMagicError),
    (b"TBT1" + bytes([0]), ts.TruncatedFileError),
    (b"TBT1" + bytes([0, 1]) + struct.pack("<Q", 4) + bytes(12), ts.TruncatedFileError),
    (b"TBT1" + bytes([0, 2]) + struct.pack("<Q", 4), ts.TruncatedFileError),
    (b"TBT1" + bytes([0, 0]), ts.TruncatedFileError),
    (b"TBT1" + bytes([0, 1]) + struct.pack("<Q", 0), ts.TruncatedFileError),
    (b"TBT1" + bytes([9, 1]) + struct.pack("<Q", 1) + bytes(4), ts.UnknownDtypeError),
    (b"TBT1" + bytes([1, 1]) + struct.pack("<Q", 2) + bytes(5), ts.TensorStoreError),
])
def test_malformed_files_rejected(tmp_path, raw, err):
    p = tmp_path / "bad.tbt"
    p.write_bytes(raw)
    with pytest.raises(err):
        ts.read_tensor(p)
    with pytest.raises(err):
        ts.read_header(p)


def test_write_rejects_unsupported(tmp_path):
    with pytest.raises(ts.UnknownDtypeError):
        ts.write_tensor(np.zeros(3, np.float64), tmp_path / "x.tbt")
    with pytest.raises(ts.TensorStoreError):
        ts.write_tensor(np.zeros((), np.float32), tmp_path / "x.tbt")


def test_manifest_rules(tmp_path):
    (tmp_path / "manifest.txt").write_text("name = empty\n")
    m = ts.load_manifest(tmp_path / "manifest.txt")
    assert m.name == "empty" and m.tensors == {}
    (tmp_path / "manifest.txt").write_text(
        "name = fast\nmeta.num_steps = 3\nmeta.topk_ratio = 0.1\nmeta.quantized = false\nmeta.note = x\n")
    m = ts.load_manifest(tmp_path)
    assert m.metadata == {"num_steps": 3, "topk_ratio": 0.1, "quantized": False, "note": "x"}
    ts.write_tensor(np.ones(2, np.float32), tmp_path / "w.tbt")
    (tmp_path / "manifest.txt").write_text("tensor.layer.w = w.tbt\n")
    ts.load_manifest(tmp_path)
    (tmp_path / "w.tbt").unlink()
    with pytest.raises(ts.ManifestError, match="layer.w"):
        ts.load_manifest(tmp_path)
    ts.write_tensor(np.ones(2, np.float32), tmp_path / "w.tbt")
    (tmp_path / "manifest.txt").write_text("tensor.w = w.tbt\ntensor.w = w.tbt\n")
    with pytest.raises(ts.ManifestError, match="duplicate"):
        ts.load_manifest(tmp_path)
    for bad in ("meta.num_steps = soon\n", "meta.quantized = maybe\n", "bogus = 1\n", "no equals sign\n"):
        (tmp_path / "manifest.txt").write_text(bad)
        with pytest.raises(ts.ManifestError):
            ts.load_manifest(tmp_path)
    with pytest.raises(ts.ManifestError):
        ts.load_manifest(tmp_path / "nowhere")


def test_reference_fixtures_read_and_rewrite_byte_identical(tmp_path):
    """Files written by the reference (make_golden_tbt.py) parse here, and writing
    the same tensors back produces byte-identical files and manifest."""
    for kind in ("float", "quantized"):
        m = ts.load_manifest(os.path.join(GOLD, kind))
        assert m.name == "toy" and m.metadata["num_layers"] == 1
        tensors = m.load_all()
        out = ts.write_manifest(tmp_path / kind, tensors, metadata=m.metadata, name=m.name)
        assert (tmp_path / kind / "manifest.txt").read_bytes() == open(
            os.path.join(GOLD, kind, "manifest.txt"), "rb").read()
        for p, path in m.tensors.items():
            assert out.tensors[p].read_bytes() == path.read_bytes(), p
    q = ts.load_manifest(os.path.join(GOLD, "quantized"))
    assert q.metadata["quantized"] is True and q.metadata["block"] == 128
    assert q.load("layers.0.qkv.q").dtype == np.int8


def test_unpack_blockquantized_host():
    from paper_2512_16093_b200.blockquant import unpack_blockquantized
    m = ts.load_manifest(os.path.join(GOLD, "quantized"))
    bq = unpack_blockquantized(m, "layers.0.qkv", 128)
    assert (bq.rows, bq.cols, bq.block) == (32, 96, 128)
    assert np.array_equal(bq.q, m.load("layers.0.qkv.q"))
    assert np.array_equal(bq.scales, m.load("layers.0.qkv.scales"))
    with pytest.raises(KeyError):
        unpack_blockquantized(m, "layers.0.nothing", 128)


@pytest.mark.gpu
def test_device_loader_streams_bit_identical(tmp_path, monkeypatch):
    import torch
    monkeypatch.setattr(ts, "_STAGE_BYTES", 1 << 20)     # force multi-chunk streaming
    monkeypatch.setattr(ts, "_stage_cache", {})
    rng = np.random.default_rng(3)
    f = rng.standard_normal((1031, 1537)).astype(np.float32)         # 6.3 MB, ragged last chunk
    c = rng.integers(-127, 128, (2304, 1200)).astype(np.int8)
    ts.write_tensor(f, tmp_path / "f.tbt")
    ts.write_tensor(c, tmp_path / "c.tbt")
    fd = ts.read_tensor_device(tmp_path / "f.tbt")
    cd = ts.read_tensor_device(tmp_path / "c.tbt")
    ct = ts.read_tensor_device(tmp_path / "c.tbt", layout="kmajor_t")
    torch.cuda.synchronize()
    assert fd.is_cuda and fd.dtype == torch.float32
    assert np.array_equal(fd.cpu().numpy().view(np.uint32), f.view(np.uint32))
    assert np.array_equal(cd.cpu().numpy(), c)
    assert np.array_equal(ct.cpu().numpy(), c.T)
    with pytest.raises(ts.TensorStoreError):
        ts.read_tensor_device(tmp_path / "f.tbt", layout="kmajor_t")


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["float", "quantized"])
def test_model_from_manifest_device_matches_reference(kind):
    """A reference-written manifest loaded straight to the device runs the same
    model as the host-loaded one (bit-identical) and matches the reference's
    own forward (tolerance: the reference is f32 numpy)."""
    import torch
    from paper_2512_16093_b200 import sampler
    from paper_2512_16093_b200.attention import error_metrics, rel_l1
    m = ts.load_manifest(os.path.join(GOLD, kind))
    ref = np.load(os.path.join(GOLD, "forward.npz"))
    host = sampler.model_from_manifest(m)
    dev = sampler.model_from_manifest(m, device=True)
    if kind == "quantized":
        w = dev.layers[0].qkv
        assert w._dev_qt.is_cuda and tuple(w._dev_qt.shape) == (96, 32)
    x = ref["x"]
    a, b = host(x, 1.0), dev(x, 1.0)
    torch.cuda.synchronize()
    assert np.array_equal(a, b)
    cos, _ = error_metrics(b, ref[kind])
    assert cos >= 0.999 and rel_l1(b, ref[kind]) <= 1e-2
    sched = sampler.schedule_from_manifest(m)
    assert sched.num_steps == 3
