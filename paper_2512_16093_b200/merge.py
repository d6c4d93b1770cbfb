"""Drop-in for ``turbobench.merge`` (/root/reference/pkg/src/turbobench/merge.py),
plus the SURVEY §8 f4 deployment path: merge delta checkpoints on the device and
block-quantize the merged projections straight into the W8A8 GEMM layout.

A delta is the elementwise f32 ``finetuned - base`` (merge.py:40-49); merging
adds ``f32(c) * delta`` onto the base in list order with numpy's two roundings
(merge.py:52-71) -- ``tb_axpy_rn`` reproduces that bit-for-bit.  Validation
(parameter sets, shapes, coefficient count) happens before any device work and
raises :class:`MergeError` with the reference's messages.
"""
from __future__ import annotations

from dataclasses import dataclass
from pathlib import Path

import numpy as np
import torch

from . import ops
from .tensor_store import ModelManifest, read_tensor_device, write_manifest


class MergeError(Exception):
    """merge.py:21."""


@dataclass
class WeightDelta:
    """Per-parameter f32 update tensors, shape-matched to the base (merge.py:25-29)."""

    entries: dict


def _shape(t):
    return tuple(t.shape)


def _check_same_params(a: dict, b: dict, what: str) -> None:
    """merge.py:32-42."""
    if a.keys() != b.keys():
        only_a = sorted(a.keys() - b.keys())
        only_b = sorted(b.keys() - a.keys())
        raise MergeError(f"{what}: parameter sets differ (extra: {only_a}, missing: {only_b})")
    for name in a:
        if _shape(a[name]) != _shape(b[name]):
            raise MergeError(f"{what}: shape mismatch for {name!r}: {_shape(a[name])} vs {_shape(b[name])}")


def extract_delta(finetuned: ModelManifest, base: ModelManifest) -> WeightDelta:
    """merge.py:45-52: elementwise ``finetuned - base`` (one f32 rounding)."""
    ft = finetuned.load_all()
    bs = base.load_all()
    _check_same_params(ft, bs, "extract_delta")
    return WeightDelta(entries={name: np.asarray(ft[name], np.float32) - np.asarray(bs[name], np.float32)
                                for name in sorted(ft)})


def _device():
    return torch.device("cuda", torch.cuda.current_device())


def _dev(t) -> torch.Tensor:
    if isinstance(t, torch.Tensor):
        return t.to(_device(), torch.float32).contiguous()
    return torch.from_numpy(np.ascontiguousarray(t, np.float32)).to(_device())


def _validate(base: dict, deltas: list, coefficients) -> list:
    if coefficients is None:
        coefficients = [1.0] * len(deltas)
    if len(coefficients) != len(deltas):
        raise MergeError(f"{len(deltas)} deltas but {len(coefficients)} coefficients")
    for d in deltas:
        _check_same_params(base, d.entries, "merge_deltas")
    return list(coefficients)


def apply_deltas_device(base: dict, deltas: list, coefficients=None) -> dict:
    """``base + sum(c * delta)`` in list order on the device; returns f32 CUDA
    tensors (inputs may be numpy arrays or tensors)."""
    coefficients = _validate(base, deltas, coefficients)
    merged = {}
    for name, t in base.items():
        acc = _dev(t).clone() if isinstance(t, torch.Tensor) else _dev(t)
        for d, c in zip(deltas, coefficients):
            ops.axpy_rn(acc.view(-1), _dev(d.entries[name]).view(-1), float(np.float32(c)))
        merged[name] = acc
    return merged


def apply_deltas(base: dict, deltas: list, coefficients=None) -> dict:
    """merge.py:55-71: pure merge, numpy in -> numpy out (computed on the device)."""
    out = apply_deltas_device(base, deltas, coefficients)
    return {name: t.cpu().numpy() for name, t in out.items()}


def merge_deltas(base: ModelManifest, deltas: list, out_dir, coefficients=None) -> ModelManifest:
    """merge.py:74-83: merge onto a base manifest and write the result."""
    merged = apply_deltas(base.load_all(), deltas, coefficients)
    return write_manifest(out_dir, merged, metadata=dict(base.metadata), name=base.name)


def merge_quantize_device(base: ModelManifest, deltas: list, coefficients=None, block: int = 128,
                          exclude=()) -> dict:
    """Deployment path: the base streams from disk into HBM
    (tensor_store.read_tensor_device), the deltas are merged there, and every
    2-D parameter not matched by ``exclude`` is block-quantized on the device
    (codes and scales bit-exact to ``quantize_blockwise`` of the host-merged
    matrix).  Returns name -> BlockQuantized (matrices, device-resident) or
    f32 CUDA tensor (vectors, excluded matrices)."""
    from .blockquant import BlockQuantConfig, quantize_blockwise
    names = sorted(base.tensors)
    coefficients = _validate({n: _Shaped(base, n) for n in names}, deltas, coefficients)
    cfg = BlockQuantConfig(block=block)
    out = {}
    for n in names:
        acc = read_tensor_device(base.tensors[n]).float()
        for d, c in zip(deltas, coefficients):
            ops.axpy_rn(acc.view(-1), _dev(d.entries[n]).view(-1), float(np.float32(c)))
        if acc.dim() == 2 and not any(p in n for p in exclude):
            out[n] = quantize_blockwise(acc, cfg)
        else:
            out[n] = acc
    return out


class _Shaped:
    """Shape-only view of a manifest entry (validation without reading the payload)."""

    def __init__(self, manifest: ModelManifest, name: str):
        from .tensor_store import read_header
        self.shape = read_header(manifest.tensors[name]).shape
