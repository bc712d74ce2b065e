"""Scattering-transfer operators (path b): data model.

Reference data model (transfer.py:50-93): per PCA term k a
``TransferOperator`` in CSC over retained w0 columns (cols, colptr, rowidx
into the w1 flat domain, vals), grouped in a ``CompressedTransfer``.

Device form (``DeviceTransfer``): one tile-major CSR per k — ``rowptr``
(K, N+1) absolute offsets, ``cols`` u32 TILE-MAJOR w0 ids ascending within a
row, ``vals`` f32, 8 bytes per stored coefficient as in the reference
container (container.py:87-88). Tile-major = tile * 4^L + local, so every
2^L x 2^L spatial tile owns a contiguous block of 4^L rows (the L-level
inverse Haar is tile-local). The frame kernels read rearranged copies built
from it (layout.py).

``DeviceTransfer.from_reference`` is the bridge from reference-format
operators (e.g. a PRTS1 container) to the device form;
``precompute.precompute_compressed`` builds it on the GPU directly.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch


@dataclass
class TransferOperator:
    """Reference-format operator (transfer.py:50-71)."""

    cols: np.ndarray
    colptr: np.ndarray
    rowidx: np.ndarray
    vals: np.ndarray
    kept_energy: float = 0.0
    total_energy: float = 0.0
    step1_entries: int = 0

    @property
    def nnz(self) -> int:
        return int(self.rowidx.size)

    def apply(self, x_idx: np.ndarray, x_val: np.ndarray, out_len: int) -> np.ndarray:
        """transfer.py:66-71: the operator applied to a sparse spectrum, on the
        GPU (kernels_b200.csc_apply: bitwise the reference's csc_apply)."""
        from .kernels_b200 import csc_apply

        return csc_apply(self.cols, self.colptr, self.rowidx, self.vals,
                         np.ascontiguousarray(x_idx, np.uint32),
                         np.ascontiguousarray(x_val, np.float64), out_len)


def flat_to_tile_major(flat, side: int, levels: int) -> np.ndarray:
    """Global Mallat flat index -> tile-major index (vectorised mirror of
    csrc/sss_common.cuh:global_to_tile)."""
    flat = np.asarray(flat, dtype=np.int64)
    r, c = flat // side, flat % side
    T = 1 << levels
    hg = np.full(flat.shape, side >> levels, np.int64)
    hl = np.ones(flat.shape, np.int64)
    done = np.zeros(flat.shape, bool)
    for lvl in range(1, levels + 1):
        h = side >> lvl
        hit = ~done & ((r >= h) | (c >= h))
        hg[hit] = h
        hl[hit] = T >> lvl
        done |= hit
    pr = np.where(r >= hg, r - hg, r)
    pc = np.where(c >= hg, c - hg, c)
    tr, tc = pr // hl, pc // hl
    lr = np.where(r >= hg, hl, 0) + pr % hl
    lc = np.where(c >= hg, hl, 0) + pc % hl
    return (tr * (side // T) + tc) * T * T + lr * T + lc


def tile_major_to_flat(side: int, levels: int) -> np.ndarray:
    """perm[t] = flat index of tile-major position t."""
    inv = flat_to_tile_major(np.arange(side * side), side, levels)
    perm = np.empty_like(inv)
    perm[inv] = np.arange(side * side)
    return perm


@dataclass
class DeviceTransfer:
    """K operators resident in HBM as tile-major CSR (canonical form)."""

    K: int
    side: int
    levels: int
    rowptr: torch.Tensor  # int64 (K, N+1), absolute offsets
    cols: torch.Tensor  # int32 (nnz,) tile-major w0 ids (u32 on the device)
    vals: torch.Tensor  # float32 (nnz,)
    nnz_per_k: list
    step1_keep: float = 0.0
    step2_fraction: float = 0.0
    kept_energy: list = None
    total_energy: list = None
    step1_entries: list = None
    # (K, ceil(N / 32)) int32 bitmaps of each term's step-1 union over flat w0
    # ids (transfer.py:233-246), when known: union columns whose step-2 energy
    # cut kept nothing are still columns of the reference operator
    unions: torch.Tensor = None

    @property
    def n(self) -> int:
        return self.side * self.side

    @property
    def nnz(self) -> int:
        return int(sum(self.nnz_per_k))

    @property
    def domain_size(self) -> int:
        return self.n

    @property
    def nbytes(self) -> int:
        """Stored bytes of the canonical operator (8 B / coefficient + row
        pointers)."""
        return self.nnz * 8 + self.rowptr.numel() * 8

    @classmethod
    def from_reference(cls, operators, side: int, levels: int, device="cuda",
                       step1_keep=0.0, step2_fraction=0.0) -> "DeviceTransfer":
        """CSC (reference TransferOperator list, flat w0 cols / w1 rows) ->
        tile-major CSR (the PRTS1 bridge direction reference -> B200)."""
        n = side * side
        f2t = flat_to_tile_major(np.arange(n), side, levels)
        rowptrs, cols_all, vals_all, nnz = [], [], [], []
        base = 0
        for op in operators:
            counts = np.diff(np.asarray(op.colptr, np.int64))
            ecol = f2t[np.repeat(np.asarray(op.cols, np.int64), counts)]
            erow = flat_to_tile_major(np.asarray(op.rowidx, np.int64), side, levels)
            order = np.lexsort((ecol, erow))
            rc = np.bincount(erow, minlength=n)
            rp = np.zeros(n + 1, np.int64)
            np.cumsum(rc, out=rp[1:])
            rowptrs.append(rp + base)
            cols_all.append(ecol[order].astype(np.uint32))
            vals_all.append(np.asarray(op.vals)[order].astype(np.float32))
            nnz.append(int(counts.sum()))
            base += int(counts.sum())
        cols = np.concatenate(cols_all) if cols_all else np.empty(0, np.uint32)
        vals = np.concatenate(vals_all) if vals_all else np.empty(0, np.float32)
        return cls(
            K=len(operators), side=side, levels=levels,
            rowptr=torch.as_tensor(np.stack(rowptrs), device=device),
            cols=torch.as_tensor(cols.view(np.int32), device=device),
            vals=torch.as_tensor(vals, device=device),
            nnz_per_k=nnz, step1_keep=step1_keep, step2_fraction=step2_fraction,
            kept_energy=[getattr(o, "kept_energy", 0.0) for o in operators],
            total_energy=[getattr(o, "total_energy", 0.0) for o in operators],
            step1_entries=[getattr(o, "step1_entries", 0) for o in operators],
        )

    def to_reference(self):
        """Device layout -> reference CSC operators (flat ids, vals f32 -> f64),
        for the PRTS1 bridge and parity checks."""
        perm = tile_major_to_flat(self.side, self.levels)
        rp = self.rowptr.cpu().numpy()
        n = self.n
        dev = self.rowptr.device
        ops = []
        if dev.type == "cuda":  # the CSR -> CSC transpose on the device (torch sort)
            perm_d = torch.as_tensor(perm, device=dev)
            cols_d = perm_d[self.cols.long() & 0xFFFFFFFF]
        else:
            cols = perm[self.cols.cpu().numpy().view(np.uint32).astype(np.int64)]
            vals = self.vals.cpu().numpy()
        for k in range(self.K):
            lo, hi = int(rp[k, 0]), int(rp[k, -1])
            if dev.type == "cuda":
                counts = self.rowptr[k, 1:] - self.rowptr[k, :-1]
                r_d = perm_d[torch.repeat_interleave(torch.arange(n, device=dev), counts)]
                c_d = cols_d[lo:hi]
                order = torch.argsort(c_d * n + r_d)
                c = c_d[order].cpu().numpy()
                r = r_d[order].cpu().numpy()
                v = self.vals[lo:hi][order].cpu().numpy()
                del counts, r_d, c_d, order
            else:
                counts = np.diff(rp[k])
                rows_tm = np.repeat(np.arange(n), counts)
                c, v, r = cols[lo:hi], vals[lo:hi], perm[rows_tm]
                order = np.lexsort((r, c))
                c, v, r = c[order], v[order], r[order]
            if self.unions is not None:  # every union column, empty spans included
                bits = np.unpackbits(self.unions[k].cpu().numpy().view(np.uint8),
                                     bitorder="little")[:n]
                ucols = np.flatnonzero(bits)
                colptr = np.searchsorted(c, np.append(ucols, n), side="left").astype(np.int64)
                colptr[-1] = c.size
            else:
                ucols, start = np.unique(c, return_index=True)
                colptr = np.append(start, c.size).astype(np.int64)
            ops.append(TransferOperator(
                cols=ucols.astype(np.uint32), colptr=colptr, rowidx=r.astype(np.uint32),
                vals=v.astype(np.float64),
                kept_energy=(self.kept_energy or [0.0] * self.K)[k],
                total_energy=(self.total_energy or [0.0] * self.K)[k],
                step1_entries=(self.step1_entries or [0] * self.K)[k]))
        return ops
