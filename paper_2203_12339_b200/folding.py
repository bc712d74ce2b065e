"""Visibility precompute and ambient folding:
`precompute_visibility` and `fold_visibility` (reference transfer.py:368-451)
on the GPU, and the folded ambient term of a frame (runtime.py:146-149).

The reference lights an environment ("ambient" light of a LightRig) through
per-k folded operators F_k = T_k v~ that take the environment's w2 (per-face
Haar) coefficients straight to w1 response coefficients, where
v~ = w0(w2(W)) and W = V F_t(eta, cos+) cos+ dw carries the binary
visibility V of every sample toward every cubemap texel. Here:

* V: `sss_visibility`, one shadow ray per (direction, sample) through the
  scene BVH (shadows.build_bvh), stored (D, N) u8;
* W and its w2 Haar: `sss_fold_weights`; the w0 Haar over samples:
  `sss_haar2d` batched over the D direction images; a permuting transpose
  puts v~ in the operator's tile-major column space;
* F_k: `sss_fold_spmm` over the frame-layout operator (the reference forms
  the dense `dense @ v_tilde[cols]`); `sss_fold_select` (compress_energy per
  direction column, exact radix cut) and `sss_fold_emit` (CSC, rows
  ascending) compress it;
* per frame: `sss_fold_apply` adds F_k L^{w2} into v_k.

No CPU fallback: every step is a kernel of the C ABI.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .lighting import face_directions, face_solid_angles
from .shadows import build_bvh, grid_triangles
from .transfer import TransferOperator, tile_major_to_flat

FOLD_FRACTION = 0.9999  # transfer.py:35 DEFAULT_FOLD_FRACTION
FACE_SIDE = 16          # precompute_visibility default (transfer.py:369)


@dataclass
class DeviceVisibility:
    """Binary visibility (D, N) u8 on the device (the reference's
    VisibilityMatrix.matrix is its (N, D) transpose)."""

    vis: torch.Tensor
    face_side: int

    @property
    def direction_count(self) -> int:
        return 6 * self.face_side * self.face_side

    def matrix(self) -> np.ndarray:
        """The reference layout: (N, D) float64 in {0, 1}."""
        return self.vis.t().cpu().numpy().astype(np.float64)


@dataclass
class DeviceFolded:
    """Folded ambient operators in HBM: per k a CSC over the D directions
    (colptr (K, D + 1) absolute, rows = flat w1 ids ascending, vals f32)."""

    K: int
    side: int
    levels: int
    face_side: int
    eta: float
    fraction: float
    colptr: torch.Tensor   # int64 (K, D + 1)
    rows: torch.Tensor     # int32 (nnz,) flat w1 ids (u32 on the device)
    vals: torch.Tensor     # float32 (nnz,)
    kept_energy: list
    total_energy: list
    step1_entries: list

    @property
    def n(self) -> int:
        return self.side * self.side

    @property
    def direction_count(self) -> int:
        return 6 * self.face_side * self.face_side

    def to_reference(self):
        """Reference FoldedTransfer operators (transfer.py:441-451): only the
        directions that kept entries are columns; vals f32 -> f64."""
        cp = self.colptr.cpu().numpy()
        rows = self.rows.cpu().numpy().view(np.uint32)
        vals = self.vals.cpu().numpy().astype(np.float64)
        ops = []
        for k in range(self.K):
            counts = np.diff(cp[k])
            cols = np.flatnonzero(counts).astype(np.uint32)
            lo, hi = int(cp[k, 0]), int(cp[k, -1])
            colptr = np.concatenate([[0], np.cumsum(counts[cols])]).astype(np.int64)
            ops.append(TransferOperator(cols=cols, colptr=colptr, rowidx=rows[lo:hi].copy(),
                                        vals=vals[lo:hi].copy(), kept_energy=self.kept_energy[k],
                                        total_energy=self.total_energy[k],
                                        step1_entries=self.step1_entries[k]))
        return ops


def _maps(side: int, levels: int, device):
    tm2flat = tile_major_to_flat(side, levels).astype(np.int64)
    flat2tm = np.empty_like(tm2flat)
    flat2tm[tm2flat] = np.arange(tm2flat.size)
    t = lambda a: torch.as_tensor(a.astype(np.int32), device=device)
    return t(tm2flat), t(flat2tm)


def _bvh_device(geometry, device):
    bvh = build_bvh(np.asarray(geometry.positions, np.float64), grid_triangles(geometry.side))
    nodes, tris = bvh.packed()
    return (torch.as_tensor(nodes, device=device), torch.as_tensor(tris, device=device),
            bvh.ray_offset, bvh.bbox_diagonal)


def precompute_visibility(geometry, face_side: int = FACE_SIDE, bvh=None,
                          device="cuda") -> DeviceVisibility:
    """precompute_visibility (transfer.py:368-391) on the GPU. `bvh` = the
    (nodes, tris, ray_offset, bbox_diagonal) tuple of a prior call, or None."""
    nodes, tris, off, diag = bvh if bvh is not None else _bvh_device(geometry, device)
    n = geometry.side * geometry.side
    d = 6 * face_side * face_side
    pos = torch.as_tensor(np.ascontiguousarray(geometry.positions, np.float32), device=device)
    nrm = torch.as_tensor(np.ascontiguousarray(geometry.normals, np.float32), device=device)
    dirs = torch.as_tensor(face_directions(face_side).reshape(-1, 3), device=device)
    vis = torch.empty((d, n), dtype=torch.uint8, device=device)
    _lib.call("sss_visibility", n, _lib.ptr(pos), _lib.ptr(nrm), d, _lib.ptr(dirs), off,
              4.0 * diag + 1.0, _lib.ptr(nodes), _lib.ptr(tris), _lib.ptr(vis), _lib.stream_ptr())
    return DeviceVisibility(vis=vis, face_side=face_side)


def fold_visibility(transfer, vis: DeviceVisibility, geometry, eta: float,
                    fraction: float = FOLD_FRACTION, device="cuda") -> DeviceFolded:
    """fold_visibility (transfer.py:394-451) for a DeviceTransfer."""
    if not 0.0 <= fraction <= 1.0:
        raise ValueError("fraction must be in [0, 1]")
    n = transfer.n
    if vis.vis.shape[1] != n or geometry.side * geometry.side != n:
        raise ValueError("visibility and samples disagree on the sample count")
    s, L = transfer.side, transfer.levels
    fs = vis.face_side
    d = vis.direction_count
    sp = _lib.stream_ptr()
    tm2flat, flat2tm = _maps(s, L, device)
    nrm = torch.as_tensor(np.ascontiguousarray(geometry.normals, np.float32), device=device)
    dirs = torch.as_tensor(face_directions(fs).reshape(-1, 3), device=device)
    dom = torch.as_tensor(np.ascontiguousarray(face_solid_angles(fs).reshape(-1)), device=device)
    w2 = torch.empty((d, n), dtype=torch.float64, device=device)
    _lib.call("sss_fold_weights", _lib.ptr(nrm), n, _lib.ptr(dirs), _lib.ptr(dom), fs,
              _lib.ptr(vis.vis), float(eta), _lib.ptr(w2), sp)
    v0 = torch.empty_like(w2)
    _lib.call("sss_haar2d", _lib.ptr(w2), _lib.ptr(v0), d, s, L, 0, sp)
    vt = w2.view(n, d)  # reuse: (N tm, D) = v0 (D, N flat) transposed + permuted
    _lib.call("sss_transpose_f64", _lib.ptr(v0), d, n, _lib.ptr(tm2flat), _lib.ptr(vt), sp)
    F = v0.view(n, d)  # v0 is dead after the transpose
    FT = torch.empty((d, n), dtype=torch.float64, device=device)
    col_t = torch.empty(d, dtype=torch.int64, device=device)
    col_fmax = torch.empty(d, dtype=torch.int32, device=device)
    col_cnt = torch.empty(d, dtype=torch.int32, device=device)
    col_e = torch.empty((d, 2), dtype=torch.float64, device=device)
    col_nz = torch.empty(d, dtype=torch.int32, device=device)
    K = transfer.K
    colptr = torch.zeros((K, d + 1), dtype=torch.int64, device=device)
    parts_rows, parts_vals = [], []
    kept, total, nzs = [], [], []
    base = 0
    for k in range(K):
        rp = transfer.rowptr[k]
        _lib.call("sss_fold_spmm", n, d, _lib.ptr(rp), _lib.ptr(transfer.cols),
                  _lib.ptr(transfer.vals), _lib.ptr(vt), _lib.ptr(F), sp)
        _lib.call("sss_transpose_f64", _lib.ptr(F), n, d, None, _lib.ptr(FT), sp)
        _lib.call("sss_fold_select", _lib.ptr(FT), n, d, float(fraction), _lib.ptr(tm2flat),
                  _lib.ptr(col_t), _lib.ptr(col_fmax), _lib.ptr(col_cnt), _lib.ptr(col_e),
                  _lib.ptr(col_nz), sp)
        cnt = col_cnt.to(torch.int64)
        cp = torch.zeros(d + 1, dtype=torch.int64, device=device)
        torch.cumsum(cnt, 0, out=cp[1:])
        nnz = int(cp[-1])
        rows = torch.empty(max(nnz, 1), dtype=torch.int32, device=device)
        vals = torch.empty(max(nnz, 1), dtype=torch.float32, device=device)
        if nnz:
            _lib.call("sss_fold_emit", _lib.ptr(FT), n, d, _lib.ptr(flat2tm), _lib.ptr(col_t),
                      _lib.ptr(col_fmax), _lib.ptr(col_cnt), _lib.ptr(cp), _lib.ptr(rows),
                      _lib.ptr(vals), sp)
        parts_rows.append(rows[:nnz])
        parts_vals.append(vals[:nnz])
        colptr[k] = cp + base
        base += nnz
        e = col_e.cpu().numpy()
        kept.append(float(e[:, 0].sum()))
        total.append(float(e[:, 1].sum()))
        nzs.append(int(col_nz.to(torch.int64).sum()))
    rows = torch.cat(parts_rows) if base else torch.zeros(1, dtype=torch.int32, device=device)
    vals = torch.cat(parts_vals) if base else torch.zeros(1, dtype=torch.float32, device=device)
    out = DeviceFolded(K=K, side=s, levels=L, face_side=fs, eta=float(eta),
                       fraction=float(fraction), colptr=colptr, rows=rows, vals=vals,
                       kept_energy=kept, total_energy=total, step1_entries=nzs)
    if out.n % 32 == 0:
        row_layout(out)  # the per-frame apply's layout, built before any graph capture
    return out


def row_layout(folded: DeviceFolded):
    """Row-major, ELL-interleaved copy of the folded CSC (built once, on the
    device; see sss_fold_apply_rows): per 32-row group g = k * (N / 32) +
    row / 32, slot-major entries (entry s of lane j at gbase[g] + 32 s + j),
    ascending by direction within a row — the per-row order csc_apply
    accumulates in — padded with (dir 0, val 0) to the group's longest row."""
    if getattr(folded, "_rows_layout", None) is not None:
        return folded._rows_layout
    n, d, K = folded.n, folded.direction_count, folded.K
    dev = folded.colptr.device
    cp = folded.colptr
    nnz = int(cp[-1, -1]) if K else 0
    kk = torch.repeat_interleave(torch.arange(K, device=dev), (cp[:, -1] - cp[:, 0]))
    dd = torch.cat([torch.repeat_interleave(torch.arange(d, device=dev), torch.diff(cp[k]))
                    for k in range(K)]) if nnz else torch.zeros(0, dtype=torch.int64, device=dev)
    rr = folded.rows[:nnz].to(torch.int64) & 0xFFFFFFFF
    krow = kk * n + rr
    order = torch.argsort(krow * d + dd, stable=True)
    krow, dd = krow[order], dd[order]
    vv = folded.vals[:nnz][order]
    counts = torch.bincount(krow, minlength=K * n)
    start = torch.zeros(K * n + 1, dtype=torch.int64, device=dev)
    torch.cumsum(counts, 0, out=start[1:])
    slot = torch.arange(nnz, device=dev) - start[krow]          # rank within the row
    width = counts.view(-1, 32).amax(1)                          # per group
    gbase = torch.zeros(width.numel() + 1, dtype=torch.int64, device=dev)
    torch.cumsum(width * 32, 0, out=gbase[1:])
    total = int(gbase[-1])
    pos = gbase[krow // 32] + slot * 32 + (krow % 32)
    ent = torch.zeros((max(total, 1), 2), dtype=torch.int32, device=dev)  # (dir, f32 bits)
    ent[pos, 0] = dd.to(torch.int32)
    ent[pos, 1] = vv.contiguous().view(torch.int32)
    folded._rows_layout = (gbase, ent)
    return folded._rows_layout


def fold_apply(folded: DeviceFolded, union_idx, union_lc, n_union, vk, stream=None,
               layout: str = "rows"):
    """vk (K, 3, N tm) += folded ambient response (runtime.py:146-149); the
    union arrays are sss_env_project's (device). layout "rows" (default):
    thread per (k, row) over the row-major copy; "csc": per row block over
    the CSC columns (the first form; same bits)."""
    _, flat2tm = _maps(folded.side, folded.levels, vk.device) if not hasattr(folded, "_flat2tm") \
        else (None, folded._flat2tm)
    folded._flat2tm = flat2tm
    if layout == "rows" and 24 * folded.direction_count <= 200 * 1024 and folded.n % 32 == 0:
        gbase, ent = row_layout(folded)
        _lib.call("sss_fold_apply_rows", folded.K, folded.n, folded.direction_count,
                  _lib.ptr(gbase), _lib.ptr(ent), _lib.ptr(union_idx),
                  _lib.ptr(union_lc), _lib.ptr(n_union), _lib.ptr(flat2tm), _lib.ptr(vk),
                  _lib.stream_ptr(stream))
        return
    _lib.call("sss_fold_apply", folded.K, folded.n, folded.direction_count,
              _lib.ptr(folded.colptr), _lib.ptr(folded.rows), _lib.ptr(folded.vals),
              _lib.ptr(union_idx), _lib.ptr(union_lc), _lib.ptr(n_union), _lib.ptr(flat2tm),
              _lib.ptr(vk), _lib.stream_ptr(stream))
