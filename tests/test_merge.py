"""Delta extraction / merging: the reference's algebra tests
(tests/test_merge.py in the reference) restated against this package -- merge
arithmetic on the device, bit-exact to the numpy elementwise order -- plus the
merge -> quantize deployment path."""
import numpy as np
import pytest

from paper_2512_16093_b200.merge import (MergeError, WeightDelta, apply_deltas, extract_delta, merge_deltas,
                                         merge_quantize_device)
from paper_2512_16093_b200.tensor_store import write_manifest


def random_tensors(seed, shapes=None):
    rng = np.random.default_rng(seed)
    shapes = shapes or {"attn.w": (24, 16), "mlp.w": (16, 48), "gain": (16,)}
    return {n: rng.standard_normal(s).astype(np.float32) for n, s in shapes.items()}


@pytest.fixture
def base(tmp_path):
    t = random_tensors(1)
    return write_manifest(tmp_path / "base", t, name="base"), t


# ------------------------------------------------------------------ host (CPU)

def test_extract_delta_identity_and_zero_base(tmp_path, base):
    manifest, tensors = base
    same = write_manifest(tmp_path / "same", tensors, name="same")
    for t in extract_delta(same, manifest).entries.values():
        assert np.array_equal(t, np.zeros_like(t))
    zeros = write_manifest(tmp_path / "zero", {k: np.zeros_like(v) for k, v in tensors.items()}, name="zero")
    d = extract_delta(manifest, zeros)
    for n, t in tensors.items():
        assert np.array_equal(d.entries[n], t)


def test_validation_errors_precede_device_work(tmp_path, base):
    manifest, tensors = base
    with pytest.raises(MergeError, match="parameter sets differ"):
        apply_deltas(manifest.load_all(), [WeightDelta({"unknown": np.zeros((2, 2), np.float32)})])
    bad = {k: v.copy() for k, v in tensors.items()}
    bad["mlp.w"] = np.zeros((2, 2), np.float32)
    with pytest.raises(MergeError, match="mlp.w"):
        apply_deltas(manifest.load_all(), [WeightDelta(bad)])
    with pytest.raises(MergeError):
        apply_deltas(manifest.load_all(), [WeightDelta(random_tensors(11))], coefficients=[1.0, 2.0])
    other = write_manifest(tmp_path / "other", {"x": np.ones(3, np.float32)}, name="o")
    with pytest.raises(MergeError, match="extract_delta"):
        extract_delta(other, manifest)
    with pytest.raises(MergeError, match="parameter sets differ"):
        merge_quantize_device(manifest, [WeightDelta({"unknown": np.zeros(1, np.float32)})])


# ----------------------------------------------------------------- device (GPU)

@pytest.mark.gpu
def test_merge_matches_elementwise_oracle(base):
    manifest, tensors = base
    d1, d2 = WeightDelta(random_tensors(5)), WeightDelta(random_tensors(6))
    merged = apply_deltas(manifest.load_all(), [d1, d2], coefficients=[1.0, -0.37])
    for n in tensors:
        want = tensors[n].copy()
        for d, c in ((d1, np.float32(1.0)), (d2, np.float32(-0.37))):
            want = want + c * d.entries[n]            # numpy: RN multiply, then RN add
        assert merged[n].dtype == np.float32
        assert np.array_equal(merged[n].view(np.uint32), want.view(np.uint32))


@pytest.mark.gpu
def test_merge_roundtrip_and_identity(tmp_path, base):
    manifest, tensors = base
    tuned_t = random_tensors(3)
    tuned = write_manifest(tmp_path / "tuned", tuned_t, name="tuned")
    delta = extract_delta(tuned, manifest)
    merged = merge_deltas(manifest, [delta], tmp_path / "merged")
    for n, want in tuned_t.items():
        tol = np.spacing(np.maximum(np.abs(want), np.abs(delta.entries[n])))
        assert np.all(np.abs(merged.load(n) - want) <= tol)
    ident = merge_deltas(manifest, [], tmp_path / "ident")
    for n, t in tensors.items():
        assert np.array_equal(ident.load(n), t)
    d = WeightDelta(random_tensors(4))
    neg = WeightDelta({k: -v for k, v in d.entries.items()})
    back = apply_deltas(manifest.load_all(), [d, neg])
    for n, t in tensors.items():
        tol = np.spacing(np.maximum(np.abs(t), np.abs(d.entries[n])))
        assert np.all(np.abs(back[n] - t) <= tol)


@pytest.mark.gpu
def test_merge_quantize_device_matches_host_merge_then_quantize(tmp_path):
    """Deployment path: codes / scales of the device-merged matrix equal the
    quantization of the host (numpy-order) merge, ragged 128-blocks included."""
    from paper_2512_16093_b200.blockquant import BlockQuantized, quantize_blockwise
    shapes = {"layers.0.qkv": (300, 260), "layers.0.rms_gain": (260,)}
    t = random_tensors(21, shapes)
    manifest = write_manifest(tmp_path / "b", t, name="b")
    d = WeightDelta(random_tensors(22, shapes))
    out = merge_quantize_device(manifest, [d], coefficients=[0.25])
    host = t["layers.0.qkv"] + np.float32(0.25) * d.entries["layers.0.qkv"]
    ref = quantize_blockwise(host)
    got = out["layers.0.qkv"]
    assert isinstance(got, BlockQuantized) and got.q.is_cuda
    assert np.array_equal(got.q_numpy(), ref.q)
    assert np.array_equal(got.scales.cpu().numpy(), ref.scales)
    g = out["layers.0.rms_gain"].cpu().numpy()
    assert np.array_equal(g, t["layers.0.rms_gain"] + np.float32(0.25) * d.entries["layers.0.rms_gain"])
