"""Drop-in for ``turbobench.tensor_store`` (/root/reference/pkg/src/turbobench/tensor_store.py),
plus the SURVEY §8 f2 device path: TBT1 payloads streamed from disk through pinned
staging buffers straight into HBM, with INT8 weight codes landing in the W8A8
GEMM's K-major B layout.

TBT1 file (tensor_store.py:1-13): ``"TBT1"``, dtype byte (0 = f32, 1 = int8), rank
byte, ``rank`` little-endian u64 extents, row-major payload; size is exactly
``6 + 8*rank + itemsize*prod(dims)``.  Manifests (tensor_store.py:161-202) are
``key = value`` lines: ``name``, ``tensor.<param> = <relative path>``,
``meta.<key> = <value>`` with typed keys.

Errors keep the reference's classes (tensor_store.py:34-53) and the conditions
its tests pin (tests/test_tensor_store.py): bad magic, truncated header/payload,
unknown dtype code, trailing bytes, unsupported dtype on write, missing /
duplicate manifest entries, unparsable typed metadata.
"""
from __future__ import annotations

import os
import struct
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

MAGIC = b"TBT1"
_CODE_OF = {np.dtype(np.float32): 0, np.dtype(np.int8): 1}
_DTYPE_OF = {0: np.dtype("<f4"), 1: np.dtype(np.int8)}


class TensorStoreError(Exception):
    """tensor_store.py:34."""


class BadMagicError(TensorStoreError):
    """tensor_store.py:38."""


class TruncatedFileError(TensorStoreError):
    """tensor_store.py:42."""


class UnknownDtypeError(TensorStoreError):
    """tensor_store.py:46."""


class ManifestError(TensorStoreError):
    """tensor_store.py:50."""


# ------------------------------------------------------------------ tensor files

def _validated(t) -> np.ndarray:
    """tensor_store.py:56-63."""
    a = np.asarray(t)
    if a.dtype not in _CODE_OF:
        raise UnknownDtypeError(f"unsupported dtype {a.dtype}; TBT1 stores float32 or int8")
    if a.ndim == 0:
        raise TensorStoreError("rank-0 tensors are not supported; store shape (1,)")
    if min(a.shape) < 1:
        raise TensorStoreError(f"every axis needs length >= 1, got {a.shape}")
    return np.ascontiguousarray(a)


def _header_bytes(dtype: np.dtype, shape) -> bytes:
    return MAGIC + bytes((_CODE_OF[np.dtype(dtype)], len(shape))) + struct.pack(f"<{len(shape)}Q", *shape)


def write_tensor(t, path) -> None:
    """tensor_store.py:66-78: one write of header + payload (no silently short file)."""
    a = _validated(t)
    payload = a.astype(a.dtype.newbyteorder("<"), copy=False).tobytes()
    with open(path, "wb") as f:
        f.write(_header_bytes(a.dtype, a.shape) + payload)


@dataclass(frozen=True)
class TensorHeader:
    dtype: np.dtype
    shape: tuple
    offset: int          # payload start
    nbytes: int          # payload bytes


def read_header(path) -> TensorHeader:
    """Parse and validate a TBT1 header against the file size (the checks of
    tensor_store.py:81-120, without reading the payload)."""
    size = os.path.getsize(path)
    with open(path, "rb") as f:
        head = f.read(6)
        if len(head) < 4 or head[:4] != MAGIC:
            raise BadMagicError(f"{path}: bad magic, not a TBT1 tensor file")
        if len(head) < 6:
            raise TruncatedFileError(f"{path}: header cut short")
        code, rank = head[4], head[5]
        if code not in _DTYPE_OF:
            raise UnknownDtypeError(f"{path}: unknown dtype code {code}")
        if rank < 1:
            raise TruncatedFileError(f"{path}: rank must be >= 1")
        dims_raw = f.read(8 * rank)
    if len(dims_raw) < 8 * rank:
        raise TruncatedFileError(f"{path}: axis lengths cut short")
    shape = struct.unpack(f"<{rank}Q", dims_raw)
    if min(shape) < 1:
        raise TruncatedFileError(f"{path}: zero-length axis in header")
    dt = _DTYPE_OF[code]
    need = int(np.prod(shape, dtype=np.int64)) * dt.itemsize
    have = size - 6 - 8 * rank
    if have < need:
        raise TruncatedFileError(f"{path}: payload has {have} bytes, header declares {need}")
    if have > need:
        raise TensorStoreError(f"{path}: {have - need} trailing bytes after the payload")
    return TensorHeader(dtype=dt, shape=tuple(int(n) for n in shape), offset=6 + 8 * rank, nbytes=need)


def read_tensor(path) -> np.ndarray:
    """tensor_store.py:81-120: host ndarray (native byte order, owned copy)."""
    h = read_header(path)
    out = np.empty(h.shape, dtype=h.dtype.newbyteorder("="))
    with open(path, "rb") as f:
        f.seek(h.offset)
        f.readinto(memoryview(out.reshape(-1).view(np.uint8)))
    if h.dtype.byteorder not in ("=", "|") and not np.little_endian:   # pragma: no cover
        out.byteswap(inplace=True)
    return out


# staging: two pinned buffers so the disk read of chunk i+1 overlaps the H2D copy of chunk i
_STAGE_BYTES = 64 << 20
_stage_cache: dict = {}


def _staging(dev):
    import torch
    st = _stage_cache.get(dev)
    if st is None:
        bufs = [torch.empty(_STAGE_BYTES, dtype=torch.uint8, pin_memory=True) for _ in range(2)]
        st = (bufs, [torch.cuda.Event() for _ in range(2)], torch.cuda.Stream(dev))
        _stage_cache[dev] = st
    return st


def read_tensor_device(path, device=None, layout: str = "row"):
    """Stream a TBT1 payload into a CUDA tensor.

    The payload is read in 64 MB chunks into two pinned staging buffers and
    copied to HBM on a copy stream, so disk and PCIe overlap; the host never
    holds the whole tensor.  ``layout="kmajor_t"`` (2-D int8 weight codes
    ``[K, N]`` in the reference's ``x @ w`` layout) returns the transposed
    ``[N, K]`` codes the W8A8 GEMM consumes as its K-major B operand
    (``tb_transpose_codes``).  The result is ordered on the current stream.
    """
    import torch
    h = read_header(path)
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    tdt = torch.float32 if h.dtype.kind == "f" else torch.int8
    out = torch.empty(h.shape, dtype=tdt, device=dev)
    raw = out.view(-1).view(torch.uint8)
    bufs, evs, cs = _staging(dev)
    cs.wait_stream(torch.cuda.current_stream(dev))
    with open(path, "rb", buffering=0) as f:
        f.seek(h.offset)
        done, i = 0, 0
        while done < h.nbytes:
            n = min(_STAGE_BYTES, h.nbytes - done)
            b = i & 1
            evs[b].synchronize()                      # copy issued from this buffer two chunks ago is done
            mv = memoryview(bufs[b].numpy())[:n]
            got = 0
            while got < n:
                r = f.readinto(mv[got:])
                if not r:
                    raise TruncatedFileError(f"{path}: file shrank while reading")
                got += r
            with torch.cuda.stream(cs):
                raw[done:done + n].copy_(bufs[b][:n], non_blocking=True)
                evs[b].record(cs)
            done += n
            i += 1
    torch.cuda.current_stream(dev).wait_stream(cs)
    out.record_stream(torch.cuda.current_stream(dev))
    if layout == "kmajor_t":
        if tdt != torch.int8 or out.dim() != 2:
            raise TensorStoreError(f"{path}: kmajor_t layout needs a 2-D int8 tensor, got {h.dtype} {h.shape}")
        from . import ops
        return ops.transpose_codes(out)
    if layout != "row":
        raise ValueError(f"unknown layout {layout!r}")
    return out


# ---------------------------------------------------------------------- manifests

_TYPED_META = {"num_steps": int, "heads": int, "model_dim": int, "num_layers": int, "block": int,
               "topk_ratio": float, "boundary_sigma": float, "sigma_max": float, "sigma_min": float}


def _parse_meta(key: str, value: str):
    """tensor_store.py:127-143."""
    if key == "quantized":
        v = value.lower()
        if v in ("true", "1", "yes"):
            return True
        if v in ("false", "0", "no"):
            return False
        raise ManifestError(f"meta.quantized must be a boolean, got {value!r}")
    cast = _TYPED_META.get(key)
    if cast is None:
        return value
    try:
        return cast(value)
    except ValueError as e:
        raise ManifestError(f"meta.{key}: cannot parse {value!r}") from e


@dataclass
class ModelManifest:
    """tensor_store.py:146-158."""

    name: str
    tensors: dict
    metadata: dict = field(default_factory=dict)
    base_dir: Path = Path(".")

    def load(self, param: str) -> np.ndarray:
        if param not in self.tensors:
            raise ManifestError(f"manifest {self.name!r} has no tensor {param!r}")
        return read_tensor(self.tensors[param])

    def load_all(self) -> dict:
        return {k: read_tensor(p) for k, p in sorted(self.tensors.items())}

    def load_device(self, param: str, device=None, layout: str = "row"):
        """Device copy of one parameter (read_tensor_device)."""
        if param not in self.tensors:
            raise ManifestError(f"manifest {self.name!r} has no tensor {param!r}")
        return read_tensor_device(self.tensors[param], device, layout)


def load_manifest(path) -> ModelManifest:
    """tensor_store.py:161-202: parse, then check that every tensor file exists and
    has a valid header (the payload is not read: read_header checks the size)."""
    path = Path(path)
    if path.is_dir():
        path = path / "manifest.txt"
    if not path.is_file():
        raise ManifestError(f"manifest not found: {path}")
    base, name = path.parent, path.stem
    tensors: dict = {}
    meta: dict = {}
    for ln, line in enumerate(path.read_text(encoding="utf-8").splitlines(), 1):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        key, eq, value = line.partition("=")
        if not eq:
            raise ManifestError(f"{path}:{ln}: expected 'key = value', got {line!r}")
        key, value = key.strip(), value.strip()
        if key == "name":
            name = value
        elif key.startswith("tensor."):
            param = key[len("tensor."):]
            if not param:
                raise ManifestError(f"{path}:{ln}: empty tensor name")
            if param in tensors:
                raise ManifestError(f"{path}:{ln}: duplicate tensor {param!r}")
            tensors[param] = base / value
        elif key.startswith("meta."):
            mk = key[len("meta."):]
            meta[mk] = _parse_meta(mk, value)
        else:
            raise ManifestError(f"{path}:{ln}: unknown key {key!r}")
    for param, tp in tensors.items():
        if not tp.is_file():
            raise ManifestError(f"tensor {param!r}: missing file {tp}")
        read_header(tp)
    return ModelManifest(name=name, tensors=tensors, metadata=meta, base_dir=base)


def write_manifest(out_dir, tensors: dict, metadata: dict | None = None, name: str = "model") -> ModelManifest:
    """tensor_store.py:205-224: tensor files + manifest.txt, then reload."""
    out_dir = Path(out_dir)
    out_dir.mkdir(parents=True, exist_ok=True)
    lines = [f"name = {name}"]
    for k in sorted(metadata or {}):
        v = metadata[k]
        lines.append(f"meta.{k} = {('true' if v else 'false') if isinstance(v, bool) else v}")
    for param in sorted(tensors):
        fname = param.replace("/", "_") + ".tbt"
        t = tensors[param]
        if hasattr(t, "detach"):
            t = t.detach().cpu().numpy()
        write_tensor(t, out_dir / fname)
        lines.append(f"tensor.{param} = {fname}")
    (out_dir / "manifest.txt").write_text("\n".join(lines) + "\n", encoding="utf-8")
    return load_manifest(out_dir / "manifest.txt")
