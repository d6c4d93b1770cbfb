"""Drop-in for ``turbobench.blockquant`` (/root/reference/pkg/src/turbobench/blockquant.py).

Block-wise symmetric INT8 quantization and the W8A8 GEMM on sm_100a.  Codes
and scales are bit-exact to the reference; ``w8a8_matmul`` /
``quantized_linear_forward`` reproduce the reference promotion order
(exact integer segment, x row scale, x column scale, ascending f32 sum)
bit-for-bit on the tensor-core path.  ``BlockQuantized`` keeps the reference
fields (numpy ``q`` / ``scales``) and lazily caches the device copies the
GEMM wants (transposed K-major codes + scales), so a weight is uploaded and
transposed once.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import ops

# largest block edge whose segment sums stay exact in f32 (blockquant.py:24-26)
_F32_EXACT_BLOCK = 1040


def _device():
    return torch.device("cuda", torch.cuda.current_device())


@dataclass
class BlockQuantConfig:
    block: int = 128

    def __post_init__(self):
        if self.block < 1:
            raise ValueError(f"block must be >= 1, got {self.block}")


@dataclass
class BlockQuantized:
    """INT8 codes plus one f32 scale per block (blockquant.py:40-64)."""

    rows: int
    cols: int
    block: int
    q: object        # int8 (rows, cols): numpy, or torch CUDA tensor
    scales: object   # float32 (ceil(rows/block), ceil(cols/block))

    @property
    def num_blocks(self) -> int:
        return int(np.prod(self.scales.shape))

    def codes_f32(self) -> np.ndarray:
        cached = getattr(self, "_codes_f32", None)
        if cached is None:
            cached = np.asarray(self.q_numpy(), dtype=np.float32)
            object.__setattr__(self, "_codes_f32", cached)
        return cached

    def q_numpy(self) -> np.ndarray:
        return self.q.cpu().numpy() if isinstance(self.q, torch.Tensor) else self.q

    # device views (cached): codes [rows, cols], transposed codes [cols, rows], scales
    def device_codes(self) -> torch.Tensor:
        t = getattr(self, "_dev_q", None)
        if t is None:
            t = self.q if isinstance(self.q, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(self.q))
            t = t.to(_device()).contiguous()
            object.__setattr__(self, "_dev_q", t)
        return t

    def device_codes_t(self) -> torch.Tensor:
        t = getattr(self, "_dev_qt", None)
        if t is None:
            t = ops.transpose_codes(self.device_codes())
            object.__setattr__(self, "_dev_qt", t)
        return t

    def device_scales(self) -> torch.Tensor:
        t = getattr(self, "_dev_s", None)
        if t is None:
            s = self.scales if isinstance(self.scales, torch.Tensor) else torch.from_numpy(
                np.ascontiguousarray(self.scales, np.float32))
            t = s.to(_device()).float().contiguous()
            object.__setattr__(self, "_dev_s", t)
        return t


def _block_extents(n: int, block: int) -> list[int]:
    nb = -(-n // block)
    return [min(block, n - i * block) for i in range(nb)]


def _expand_scales(scales: np.ndarray, block: int, rows: int, cols: int) -> np.ndarray:
    """blockquant.py:72-75."""
    r = np.repeat(scales, _block_extents(rows, block), axis=0)
    return np.repeat(r, _block_extents(cols, block), axis=1)


def _block_absmax(m: np.ndarray, block: int) -> np.ndarray:
    """blockquant.py:78-88 (device max-abs per block via the quantizer's scale)."""
    q, s = ops.quantize_blockwise(torch.from_numpy(np.ascontiguousarray(m, np.float32)).to(_device()), block)
    return (s.double() * 127.0).float().cpu().numpy()


def quantize_blockwise(m, cfg: BlockQuantConfig | None = None) -> BlockQuantized:
    """blockquant.py:91-110 -- bit-exact codes and scales (tb_quantize_blockwise)."""
    cfg = cfg or BlockQuantConfig()
    as_torch = isinstance(m, torch.Tensor)
    x = m if as_torch else np.asarray(m, dtype=np.float32)
    if x.ndim != 2:
        raise ValueError(f"expected a matrix, got shape {tuple(x.shape)}")
    xd = x.to(_device()) if as_torch else torch.from_numpy(np.ascontiguousarray(x)).to(_device())
    q, s = ops.quantize_blockwise(xd, cfg.block, check_finite=True)
    if as_torch:
        return BlockQuantized(rows=x.shape[0], cols=x.shape[1], block=cfg.block, q=q, scales=s)
    bq = BlockQuantized(rows=x.shape[0], cols=x.shape[1], block=cfg.block, q=q.cpu().numpy(),
                        scales=s.cpu().numpy())
    object.__setattr__(bq, "_dev_q", q)
    object.__setattr__(bq, "_dev_s", s)
    return bq


def dequantize_blockwise(bq: BlockQuantized):
    """blockquant.py:113-116."""
    out = ops.dequantize_blockwise(bq.device_codes(), bq.device_scales(), bq.block)
    return out if isinstance(bq.q, torch.Tensor) else out.cpu().numpy()


def _exact_int_matmul(a8: np.ndarray, b8: np.ndarray) -> np.ndarray:
    """blockquant.py:119-129 (host helper kept for API parity)."""
    if a8.shape[1] <= _F32_EXACT_BLOCK:
        return a8.astype(np.float32) @ b8.astype(np.float32)
    return (a8.astype(np.int64) @ b8.astype(np.int64)).astype(np.float32)


def w8a8_matmul(a: BlockQuantized, b: BlockQuantized):
    """blockquant.py:132-161 on the tensor-core GEMM (bit-exact promotion order)."""
    if a.cols != b.rows:
        raise ValueError(f"inner dims differ: {a.cols} vs {b.rows}")
    if a.block != b.block:
        raise ValueError(f"block edges differ: {a.block} vs {b.block}")
    out = ops.w8a8_gemm(a.device_codes(), a.device_scales(), b.device_codes_t(), b.device_scales(), a.block)
    return out if isinstance(a.q, torch.Tensor) else out.cpu().numpy()


def quantized_linear_forward(x, w: BlockQuantized, bias=None, exact: bool = True, out_dtype=torch.float32):
    """blockquant.py:164-182: on-the-fly activation quantization + W8A8 + bias.

    numpy in -> numpy f32 out (bit-exact to the reference).  Torch CUDA in ->
    torch out; ``exact=False`` selects the single-FMA promotion (tolerance
    level) used by the DiT step.
    """
    as_torch = isinstance(x, torch.Tensor)
    if x.ndim != 2 or x.shape[1] != w.rows:
        raise ValueError(f"activation shape {tuple(x.shape)} does not match weight rows {w.rows}")
    xd = x if as_torch else torch.from_numpy(np.ascontiguousarray(x, np.float32)).to(_device())
    bd = None
    if bias is not None:
        bd = bias if isinstance(bias, torch.Tensor) else torch.from_numpy(np.asarray(bias, np.float32))
        bd = bd.to(_device()).float()
    y = ops.quantized_linear(xd, w.device_codes_t(), w.device_scales(), w.block, bd, out_dtype, exact,
                             check_finite=not as_torch)
    return y if as_torch else y.cpu().numpy()


def compression_ratio(bq: BlockQuantized, baseline_bytes_per_element: float) -> float:
    """blockquant.py:185-190."""
    if baseline_bytes_per_element <= 0:
        raise ValueError("baseline_bytes_per_element must be positive")
    n = bq.rows * bq.cols
    return (1 * n + 4 * bq.num_blocks) / (baseline_bytes_per_element * n)


def pack_blockquantized(bq: BlockQuantized, name: str) -> dict:
    """blockquant.py:193-195."""
    return {f"{name}.q": bq.q_numpy(), f"{name}.scales": np.asarray(
        bq.scales.cpu() if isinstance(bq.scales, torch.Tensor) else bq.scales)}


def unpack_blockquantized(manifest, name: str, block: int, device: bool = False) -> BlockQuantized:
    """blockquant.py:198-202: rebuild from the ``<name>.q`` / ``<name>.scales`` entries.

    ``device=True`` streams the codes from disk into HBM already in
    the GEMM's K-major B layout ([N, K], tensor_store.read_tensor_device) and the
    scales next to them; ``q`` is then the [K, N] view of those codes, so nothing
    is staged through a host ndarray or transposed again at first use."""
    from .tensor_store import read_tensor, read_tensor_device
    qp, sp = manifest.tensors[f"{name}.q"], manifest.tensors[f"{name}.scales"]   # KeyError, as the reference
    if not device:
        q, s = read_tensor(qp), read_tensor(sp)
        return BlockQuantized(rows=q.shape[0], cols=q.shape[1], block=block, q=q, scales=s)
    qt = read_tensor_device(qp, layout="kmajor_t")
    s = read_tensor_device(sp)
    bq = BlockQuantized(rows=qt.shape[1], cols=qt.shape[0], block=block, q=qt.t(), scales=s)
    object.__setattr__(bq, "_dev_qt", qt)
    object.__setattr__(bq, "_dev_s", s)
    return bq
