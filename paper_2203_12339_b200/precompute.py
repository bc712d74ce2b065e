"""GPU precompute (path d): the dipole pair pass and the reference's two-step
wavelet compression, producing a device-resident ``DeviceTransfer``.

Reference: ``precompute_compressed(samples, atlas, basis, step1_keep,
step2_fraction)`` (transfer.py:350-361). For a geometry image (identity
atlas) with L-level Haar on w0 and w1 (L <= 3), per PCA term k:

  1. ``sss_pair_block``  — transfer_block rows (lerp, bitwise) or the exact
     per-pair R_d projection; w0 Haar -> D (step-1 rows); f32; w1 Haar -> M.
  2. ``sss_step1_select`` — per-row top-n, union of kept w0 ids (step1_unions).
  3. ``sss_step2_select`` — per-union-column energy cut (_threshold_columns).
  4. ``sss_emit`` x2 + scans — the kept entries, straight into the tile-major
     CSR frame layout.

D and M are materialised per k (2 N^2 doubles: 69 GB at 256^2) — the B200's
180 GB replaces the reference's spill file and per-group re-evaluation. Exact
mode (per-pair R_d at every training material) runs step 1 K-fused and
streamed instead (``sss_pair_rows_exact``: R_d once per pair for all terms,
receiver-tile blocks of step-1 rows, no N^2 D).
"""

from __future__ import annotations

import math
import time

import numpy as np
import torch

from . import _lib
from .basis import DiffusionBasis, _derive
from .geometry import GeometryImage
from .transfer import DeviceTransfer, flat_to_tile_major

EMIT_CHUNK = 4096


class PrecomputeStats(dict):
    pass


def _tables(side, levels, dev):
    n = side * side
    f2t = flat_to_tile_major(np.arange(n), side, levels)
    t2f = np.empty_like(f2t)
    t2f[f2t] = np.arange(n)
    return (torch.as_tensor(f2t.astype(np.int32), device=dev),
            torch.as_tensor(t2f.astype(np.int32), device=dev))


def exact_mode_tables(basis: DiffusionBasis, eta=None):
    """(Pkm (K, M) float32, mat (M, 4) float32): b_k(r) = sum_m Pkm[k, m]
    R_d(r; sigma_m) with R_d = c_m (z_r (s + 1/d_r) e^{-s d_r} / d_r^2 + ...),
    c_m = alpha'/(4 pi). U is recovered from decompose (basisgen.py:151,
    SURVEY §8c)."""
    eta = basis.eta if eta is None else eta
    P = (basis.U / basis.singular_values[None, : basis.K]).T
    mat = []
    for sp, sa in basis.sigma_nodes:
        ap, s, z_r, z_v = _derive(sp, sa, eta)
        mat.append([s, z_r, z_v, ap / (4.0 * math.pi)])
    return np.ascontiguousarray(P, np.float32), np.ascontiguousarray(mat, np.float32)


class PairPass:
    """Device buffers + launches of the pair pass for one geometry image."""

    def __init__(self, geometry: GeometryImage, basis: DiffusionBasis, levels: int,
                 exact: bool = False, device="cuda"):
        _lib.load()
        if levels > 3:
            raise ValueError("the GPU pair pass supports levels <= 3")
        self.side, self.levels, self.exact = geometry.side, levels, exact
        self.n = geometry.count
        self.K = basis.K
        dev = torch.device(device)
        self.pos = torch.as_tensor(geometry.positions, device=dev).contiguous()
        self.area = torch.as_tensor(geometry.area, device=dev).contiguous()
        slopes = (basis.bases[:, 1:] - basis.bases[:, :-1]) / np.diff(basis.r_nodes)
        self.r_nodes = torch.as_tensor(basis.r_nodes, device=dev)
        self.bases = torch.as_tensor(np.ascontiguousarray(basis.bases), device=dev)
        self.slopes = torch.as_tensor(np.ascontiguousarray(slopes), device=dev)
        self.nr = len(basis.r_nodes)
        P, mat = exact_mode_tables(basis)
        self.Pkm = torch.as_tensor(P, device=dev)
        self.mat = torch.as_tensor(mat, device=dev)
        self.n_mat = mat.shape[0]
        self.r_max = float(basis.r_max)
        self.Pkm_host = self.mat_host = None

    def run_rows_exact(self, rt0: int, nrt: int, D, stream=None):
        """K-fused exact pass for receiver tiles [rt0, rt0 + nrt): D (K, nrt *
        4^L, N) = the step-1 rows of every term (sss_pair_rows_exact)."""
        if self.Pkm_host is None:  # host tables: the library copies them into the launch
            self.Pkm_host = self.Pkm.cpu().contiguous()
            self.mat_host = self.mat.cpu().contiguous()
        _lib.call("sss_pair_rows_exact", self.levels, self.side, _lib.ptr(self.pos),
                  _lib.ptr(self.area), self.K, _lib.ptr(self.Pkm_host), _lib.ptr(self.mat_host),
                  self.n_mat, self.r_max, rt0, nrt, _lib.ptr(D), _lib.stream_ptr(stream))

    def run(self, k: int, D=None, M=None, stream=None):
        _lib.call("sss_pair_block", self.levels, int(self.exact), self.side, _lib.ptr(self.pos),
                  _lib.ptr(self.area), _lib.ptr(self.r_nodes), _lib.ptr(self.bases),
                  _lib.ptr(self.slopes), self.nr, k, _lib.ptr(self.Pkm), _lib.ptr(self.mat),
                  self.n_mat, self.r_max, _lib.ptr(D), _lib.ptr(M), _lib.stream_ptr(stream))

    @property
    def pairs(self) -> int:
        return self.n * self.n


def precompute_compressed(geometry: GeometryImage, basis: DiffusionBasis, levels: int,
                          step1_keep: float, step2_fraction: float, exact: bool = False,
                          device="cuda", stats: dict = None) -> DeviceTransfer:
    """Build the K compressed operators on the GPU (reference API:
    transfer.precompute_compressed). Returns the frame-layout operator."""
    if not 0.0 <= step2_fraction <= 1.0:
        raise ValueError("step2_fraction must lie in [0, 1]")
    side, n, K = geometry.side, geometry.count, basis.K
    dev = torch.device(device)
    pp = PairPass(geometry, basis, levels, exact, device)
    f2t, t2f = _tables(side, levels, dev)
    n_keep = max(int(round(step1_keep * n)), 1)  # transfer.py:220
    T2 = (1 << levels) ** 2
    nchunks = (n + EMIT_CHUNK - 1) // EMIT_CHUNK
    sp = _lib.stream_ptr()
    t_start = time.perf_counter()
    # exact mode: step 1 K-fused and streamed by receiver blocks (R_d once
    # per pair for all terms); lerp mode: per term from the full D below
    exact_unions = step1_unions_exact(pp, n_keep, t2f)[0] if exact else None
    D = None if exact else torch.empty((n, n), dtype=torch.float64, device=dev)
    M = torch.empty((n, n), dtype=torch.float64, device=dev)
    union = torch.empty((n + 31) // 32, dtype=torch.int32, device=dev)
    col_t = torch.empty(n, dtype=torch.int64, device=dev)
    col_fmax = torch.empty(n, dtype=torch.int32, device=dev)
    col_cnt = torch.empty(n, dtype=torch.int32, device=dev)
    col_e = torch.empty((n, 2), dtype=torch.float64, device=dev)
    counts = torch.empty(n * nchunks, dtype=torch.int32, device=dev)
    offs = torch.empty(n * nchunks, dtype=torch.int64, device=dev)
    bsums = torch.empty((n * nchunks + 1023) // 1024 + 1, dtype=torch.int64, device=dev)
    total = torch.empty(1, dtype=torch.int64, device=dev)
    rowptr = torch.empty((K, n + 1), dtype=torch.int64, device=dev)
    cols_k, vals_k, nnz, kept_e, total_e, union_sizes, unions = [], [], [], [], [], [], []
    base = 0
    for k in range(K):
        pp.run(k, D, M)
        if exact:
            union.copy_(exact_unions[k])
        else:
            union.zero_()
            _lib.call("sss_step1_select", _lib.ptr(D), n, n, n_keep, _lib.ptr(t2f), _lib.ptr(union),
                      sp)
        _lib.call("sss_step2_select", _lib.ptr(M), n, float(step2_fraction), _lib.ptr(f2t),
                  _lib.ptr(t2f), _lib.ptr(union), _lib.ptr(col_t), _lib.ptr(col_fmax),
                  _lib.ptr(col_cnt), _lib.ptr(col_e), sp)
        _lib.call("sss_emit", 0, _lib.ptr(M), n, T2, EMIT_CHUNK, _lib.ptr(col_t), _lib.ptr(col_fmax),
                  _lib.ptr(t2f), _lib.ptr(counts), None, None, None, sp)
        _lib.call("sss_scan_u32", _lib.ptr(counts), _lib.ptr(offs), n * nchunks, _lib.ptr(bsums),
                  _lib.ptr(total), sp)
        nk = int(total.item())
        cols = torch.empty(max(nk, 1), dtype=torch.int32, device=dev)
        vals = torch.empty(max(nk, 1), dtype=torch.float32, device=dev)
        _lib.call("sss_emit", 1, _lib.ptr(M), n, T2, EMIT_CHUNK, _lib.ptr(col_t), _lib.ptr(col_fmax),
                  _lib.ptr(t2f), None, _lib.ptr(offs), _lib.ptr(cols), _lib.ptr(vals), sp)
        _lib.call("sss_rowptr", _lib.ptr(offs), nchunks, n, base, _lib.ptr(total),
                  _lib.ptr(rowptr[k]), sp)
        e = col_e.sum(dim=0).cpu().numpy()
        kept_e.append(float(e[0]))
        total_e.append(float(e[1]))
        union_sizes.append(int(np.unpackbits(union.cpu().numpy().view(np.uint8)).sum()))
        unions.append(union.clone())
        cols_k.append(cols[:nk])
        vals_k.append(vals[:nk])
        nnz.append(nk)
        base += nk
    torch.cuda.synchronize()
    del D, M
    t_total = time.perf_counter() - t_start
    dt = DeviceTransfer(
        K=K, side=side, levels=levels, rowptr=rowptr,
        cols=torch.cat(cols_k) if cols_k else torch.empty(0, dtype=torch.int32, device=dev),
        vals=torch.cat(vals_k) if vals_k else torch.empty(0, dtype=torch.float32, device=dev),
        nnz_per_k=nnz, step1_keep=step1_keep, step2_fraction=step2_fraction,
        kept_energy=kept_e, total_energy=total_e, step1_entries=[n * min(n_keep, n)] * K,
        unions=torch.stack(unions) if unions else None)
    if stats is not None:
        stats.update(seconds=t_total, union_sizes=union_sizes, nnz=nnz, n_keep=n_keep,
                     pairs=pp.pairs * K)
    return dt


def step1_unions_exact(pp: "PairPass", n_keep: int, t2f: torch.Tensor, block_bytes: int = 4 << 30,
                       stats: dict = None):
    """Step 1 of the exact mode, K-fused and streamed (BASELINE C5): receiver
    tiles in blocks whose (K, rows, N) fp64 step-1 rows fit `block_bytes`;
    per block one sss_pair_rows_exact launch (R_d once per pair, all K terms)
    and per term one sss_step1_select over the block's rows. Returns the
    per-term union bitmaps (flat w0 ids)."""
    n, K = pp.n, pp.K
    T2 = (1 << pp.levels) ** 2
    tiles = n // T2
    dev = pp.pos.device
    nrt = max(1, min(tiles, block_bytes // (K * T2 * n * 8)))
    D = torch.empty((K, nrt * T2, n), dtype=torch.float64, device=dev)
    unions = [torch.zeros((n + 31) // 32, dtype=torch.int32, device=dev) for _ in range(K)]
    sp = _lib.stream_ptr()
    t_pair = t_sel = 0.0
    for rt0 in range(0, tiles, nrt):
        nb = min(nrt, tiles - rt0)
        Db = D.view(-1)[: K * nb * T2 * n].view(K, nb * T2, n)  # a short last block packs tighter
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e[0].record()
        pp.run_rows_exact(rt0, nb, Db)
        e[1].record()
        for k in range(K):
            _lib.call("sss_step1_select", _lib.ptr(Db[k]), n, nb * T2, n_keep, _lib.ptr(t2f),
                      _lib.ptr(unions[k]), sp)
        e[2].record()
        if stats is not None:
            e[2].synchronize()
            t_pair += e[0].elapsed_time(e[1]) / 1e3
            t_sel += e[1].elapsed_time(e[2]) / 1e3
    if stats is not None:
        stats.update(pair_s=t_pair, select_s=t_sel, block_tiles=nrt, pairs=n * n)
    return unions, D


def step1_only(geometry: GeometryImage, basis: DiffusionBasis, levels: int, step1_keep: float,
               exact: bool = True, ks=None, device="cuda", stats: dict = None):
    """The C5 workload: pair pass (+ w0 Haar) and per-row top-n for each k;
    returns per-k union bitmaps (flat w0 ids). Exact mode runs K-fused and
    streamed (step1_unions_exact); lerp mode one term at a time."""
    side, n = geometry.side, geometry.count
    dev = torch.device(device)
    pp = PairPass(geometry, basis, levels, exact, device)
    _, t2f = _tables(side, levels, dev)
    n_keep = max(int(round(step1_keep * n)), 1)
    if exact and ks is None:
        return step1_unions_exact(pp, n_keep, t2f, stats=stats)
    D = torch.empty((n, n), dtype=torch.float64, device=dev)
    unions = []
    for k in (range(basis.K) if ks is None else ks):
        pp.run(k, D, None)
        u = torch.zeros((n + 31) // 32, dtype=torch.int32, device=dev)
        _lib.call("sss_step1_select", _lib.ptr(D), n, n, n_keep, _lib.ptr(t2f), _lib.ptr(u),
                  _lib.stream_ptr())
        unions.append(u)
    return unions, D
