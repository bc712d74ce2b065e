"""Wavelet transforms and exact truncation on the GPU (reference
wavelets.py:56-153 API over torch CUDA tensors).

``haar2d`` / ``haar2d_inverse`` accept (s, s) or (B, s, s) float64 CUDA
tensors and an optional level limit (default: full pyramid, i.e. the
reference's transform); ``compress_top_n`` reproduces the reference's stable
selection rule (|c| descending, ties -> lower flat index) exactly.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib


def _full_levels(side: int) -> int:
    return int(side).bit_length() - 1


def _run(grid: torch.Tensor, levels, inverse: bool) -> torch.Tensor:
    if not isinstance(grid, torch.Tensor) or not grid.is_cuda:
        raise TypeError("expected a CUDA tensor (there is no CPU path)")
    a = grid.to(torch.float64).contiguous()
    single = a.dim() == 2
    if single:
        a = a[None]
    if a.dim() != 3 or a.shape[-1] != a.shape[-2]:
        raise ValueError("expected (s, s) grid or (B, s, s) batch")
    side = a.shape[-1]
    if side < 2 or side & (side - 1):
        raise ValueError(f"grid side must be a power of two >= 2, got {side}")
    lv = _full_levels(side) if levels is None else int(levels)
    out = torch.empty_like(a)
    _lib.call("sss_haar2d", _lib.ptr(a), _lib.ptr(out), a.shape[0], side, lv, int(inverse),
              _lib.stream_ptr())
    return out[0] if single else out


def haar2d(grid, levels=None):
    """Forward L-level orthonormal Haar (full pyramid by default)."""
    return _run(grid, levels, False)


def haar2d_inverse(grid, levels=None):
    return _run(grid, levels, True)


@dataclass(frozen=True)
class SparseSpectrum:
    """wavelets.py:75-105 (indices sorted uint32, values float64)."""

    indices: np.ndarray
    values: np.ndarray
    size: int
    total_energy: float
    kept_energy: float

    @property
    def count(self) -> int:
        return int(self.indices.size)

    def to_dense(self) -> np.ndarray:
        d = np.zeros(self.size, np.float64)
        d[self.indices] = self.values
        return d


def select_top_n_device(v: torch.Tensor, n: int):
    """(B, n_dom) float64 CUDA -> (x masked (B, n_dom), mask words, energy (B, 2))."""
    v = v.to(torch.float64).contiguous()
    if v.dim() == 1:
        v = v[None]
    B, n_dom = v.shape
    x = torch.empty_like(v)
    mask = torch.empty((B, (n_dom + 31) // 32), dtype=torch.int32, device=v.device)
    energy = torch.empty((B, 2), dtype=torch.float64, device=v.device)
    _lib.call("sss_select_topn", _lib.ptr(v), B, n_dom, int(n), None, _lib.ptr(x), _lib.ptr(mask),
              _lib.ptr(energy), _lib.stream_ptr())
    return x, mask, energy


def mask_to_indices(mask_row: np.ndarray, n_dom: int) -> np.ndarray:
    bits = np.unpackbits(np.asarray(mask_row).view(np.uint8), bitorder="little")[:n_dom]
    return np.flatnonzero(bits).astype(np.uint32)


def compress_top_n(spectrum, n: int) -> SparseSpectrum:
    """Keep the n largest-magnitude coefficients (ties: lower flat index)."""
    if n < 0:
        raise ValueError("n must be >= 0")
    v = torch.as_tensor(spectrum, dtype=torch.float64).reshape(-1)
    if not v.is_cuda:
        v = v.cuda()
    x, mask, energy = select_top_n_device(v[None], min(n, v.numel()))
    idx = mask_to_indices(mask[0].cpu().numpy(), v.numel())
    vals = v.cpu().numpy()[idx]
    e = energy[0].cpu().numpy()
    return SparseSpectrum(indices=idx, values=vals, size=v.numel(), total_energy=float(e[0]),
                          kept_energy=float(e[1]))
