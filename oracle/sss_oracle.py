"""CPU oracle for the relight / material-edit hot path — TEST INFRASTRUCTURE ONLY.

This module is the checker, never the product: only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl
reference`` leg may import it. The product (``paper_2203_12339_b200``) never
imports it and has no CPU fallback.

It restates, in numpy float64, the reference's algorithm for the path named by
BASELINE.json's north star (reference = ``sssrelight`` under
/root/reference/pkg). Each function cites the reference file:line it follows.
Where BASELINE asks for something the reference does not have (L-level
Haar, a Haar w1 transform, SH light transfer, geometry images, the exact
per-pair PCA projection) the restatement is composed from the reference's own
primitives and says so.

Parity pin: ``tests/golden/make_golden.py`` imports the real reference in the
build container and writes small fixtures under ``tests/golden/``;
``tests/test_oracle_golden.py`` checks this module against them bit-for-bit
(full-pyramid Haar / 9/7, top-n, energy select, transfer rows, CSC apply, the
full two-step precompute at levels=full + w1=9/7, and the frame).

Floating-point conventions follow the reference numpy twin
(``_kernels_np.py``): no fused multiply-add, element-wise expression order
kept exactly so results are bitwise reproducible.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

# ---------------------------------------------------------------------------
# constants — _kernels_np.py:18-26
# ---------------------------------------------------------------------------
CDF97_ALPHA = -1.586134342059924
CDF97_BETA = -0.05298011857296141
_T = 1.0 + 2.0 * CDF97_BETA * (1.0 + 2.0 * CDF97_ALPHA)
CDF97_GAMMA = -(1.0 + 2.0 * CDF97_ALPHA) / (2.0 * _T)
CDF97_DELTA = 0.4435068520511142
CDF97_ZETA = math.sqrt(2.0) / _T
CDF97_INV_ZETA = 1.0 / CDF97_ZETA
ISQRT2 = 1.0 / math.sqrt(2.0)


def full_levels(side: int) -> int:
    return int(side).bit_length() - 1


# ---------------------------------------------------------------------------
# Haar — _kernels_np.py:33-74, restated with a level limit (SURVEY §8c "L-level
# Haar"): identical arithmetic and Mallat layout, stop after L levels.
# L = log2(side) reproduces haar2d_fwd_batch / haar2d_inv_batch bitwise.
# ---------------------------------------------------------------------------

def _haar_axis_fwd(a):  # _kernels_np.py:33-41
    h = a.shape[-1] // 2
    ev = a[..., 0::2]
    od = a[..., 1::2]
    lo = (ev + od) * ISQRT2
    hi = (ev - od) * ISQRT2
    a[..., :h] = lo
    a[..., h:] = hi


def _haar_axis_inv(a):  # _kernels_np.py:44-50
    h = a.shape[-1] // 2
    lo = a[..., :h].copy()
    hi = a[..., h:].copy()
    a[..., 0::2] = (lo + hi) * ISQRT2
    a[..., 1::2] = (lo - hi) * ISQRT2


def _levels_or_full(side, levels):
    full = full_levels(side)
    if levels is None:
        return full
    if not 0 <= levels <= full:
        raise ValueError(f"levels must lie in [0, {full}]")
    return levels


def haar2d_fwd(blocks, levels=None):
    """(B, s, s) forward Haar, L levels (default: full pyramid).

    Follows haar2d_fwd_batch (_kernels_np.py:53-62): per level rows, then
    columns, on the shrinking top-left s x s sub-block.
    """
    out = np.array(blocks, dtype=np.float64, copy=True)
    s = out.shape[-1]
    for _ in range(_levels_or_full(s, levels)):
        sub = out[..., :s, :s]
        _haar_axis_fwd(sub)
        _haar_axis_fwd(sub.swapaxes(-1, -2))
        s //= 2
    return out


def haar2d_inv(blocks, levels=None):
    """Exact adjoint of haar2d_fwd (haar2d_inv_batch, _kernels_np.py:65-74)."""
    out = np.array(blocks, dtype=np.float64, copy=True)
    full = out.shape[-1]
    lv = _levels_or_full(full, levels)
    s = full >> (lv - 1) if lv else full * 2
    while s <= full and lv:
        sub = out[..., :s, :s]
        _haar_axis_inv(sub.swapaxes(-1, -2))
        _haar_axis_inv(sub)
        s *= 2
    return out


# ---------------------------------------------------------------------------
# CDF 9/7 — _kernels_np.py:81-135 (kept for reference-container parity mode)
# ---------------------------------------------------------------------------

def _cdf97_axis_fwd(a):  # _kernels_np.py:81-97
    s = a.shape[-1]
    h = s // 2
    a[..., 1:s - 2:2] += CDF97_ALPHA * (a[..., 0:s - 3:2] + a[..., 2:s - 1:2])
    a[..., s - 1] += 2.0 * CDF97_ALPHA * a[..., s - 2]
    a[..., 2::2] += CDF97_BETA * (a[..., 1:s - 2:2] + a[..., 3::2])
    a[..., 0] += 2.0 * CDF97_BETA * a[..., 1]
    a[..., 1:s - 2:2] += CDF97_GAMMA * (a[..., 0:s - 3:2] + a[..., 2:s - 1:2])
    a[..., s - 1] += 2.0 * CDF97_GAMMA * a[..., s - 2]
    a[..., 2::2] += CDF97_DELTA * (a[..., 1:s - 2:2] + a[..., 3::2])
    a[..., 0] += 2.0 * CDF97_DELTA * a[..., 1]
    ev = a[..., 0::2] * CDF97_ZETA
    od = a[..., 1::2] * CDF97_INV_ZETA
    a[..., :h] = ev
    a[..., h:] = od


def _cdf97_axis_inv(a):  # _kernels_np.py:100-111
    s = a.shape[-1]
    ev = a[..., : s // 2] * CDF97_INV_ZETA
    od = a[..., s // 2:] * CDF97_ZETA
    a[..., 0::2] = ev
    a[..., 1::2] = od
    a[..., 0] -= 2.0 * CDF97_DELTA * a[..., 1]
    a[..., 2::2] -= CDF97_DELTA * (a[..., 1:s - 2:2] + a[..., 3::2])
    a[..., s - 1] -= 2.0 * CDF97_GAMMA * a[..., s - 2]
    a[..., 1:s - 2:2] -= CDF97_GAMMA * (a[..., 0:s - 3:2] + a[..., 2:s - 1:2])
    a[..., 0] -= 2.0 * CDF97_BETA * a[..., 1]
    a[..., 2::2] -= CDF97_BETA * (a[..., 1:s - 2:2] + a[..., 3::2])
    a[..., s - 1] -= 2.0 * CDF97_ALPHA * a[..., s - 2]
    a[..., 1:s - 2:2] -= CDF97_ALPHA * (a[..., 0:s - 3:2] + a[..., 2:s - 1:2])


def cdf97_fwd(blocks, levels=None):  # cdf97_fwd_batch, _kernels_np.py:114-123
    out = np.array(blocks, dtype=np.float64, copy=True)
    s = out.shape[-1]
    for _ in range(_levels_or_full(s, levels)):
        sub = out[..., :s, :s]
        _cdf97_axis_fwd(sub)
        _cdf97_axis_fwd(sub.swapaxes(-1, -2))
        s //= 2
    return out


def cdf97_inv(blocks, levels=None):  # cdf97_inv_batch, _kernels_np.py:126-135
    out = np.array(blocks, dtype=np.float64, copy=True)
    full = out.shape[-1]
    lv = _levels_or_full(full, levels)
    s = full >> (lv - 1) if lv else full * 2
    while s <= full and lv:
        sub = out[..., :s, :s]
        _cdf97_axis_inv(sub.swapaxes(-1, -2))
        _cdf97_axis_inv(sub)
        s *= 2
    return out


def w_fwd(kind, blocks, levels):
    return (haar2d_fwd if kind == "haar" else cdf97_fwd)(blocks, levels)


def w_inv(kind, blocks, levels):
    return (haar2d_inv if kind == "haar" else cdf97_inv)(blocks, levels)


# ---------------------------------------------------------------------------
# truncation — wavelets.py:108-153
# ---------------------------------------------------------------------------

@dataclass
class Spectrum:
    indices: np.ndarray  # uint32 sorted
    values: np.ndarray  # float64
    size: int
    total_energy: float
    kept_energy: float

    @property
    def count(self):
        return int(self.indices.size)

    def to_dense(self):
        d = np.zeros(self.size)
        d[self.indices] = self.values
        return d


def _make_spectrum(flat, order, kept):  # wavelets.py:116-125
    idx = np.sort(order[:kept]).astype(np.uint32)
    vals = flat[idx]
    total = float(np.sum(flat * flat))
    kept_e = min(float(np.sum(vals * vals)), total)
    return Spectrum(idx, vals, flat.size, total, kept_e)


def compress_top_n(spectrum, n: int) -> Spectrum:
    """wavelets.py:128-136: n largest |c|, stable tie -> lower flat index."""
    if n < 0:
        raise ValueError("n must be >= 0")
    flat = np.asarray(spectrum, dtype=np.float64).reshape(-1)
    n = min(n, flat.size)
    order = np.argsort(-np.abs(flat), kind="stable")
    return _make_spectrum(flat, order, n)


def compress_energy(spectrum, fraction: float) -> Spectrum:
    """wavelets.py:139-153: shortest |c|-ordered prefix reaching the fraction."""
    if not 0.0 <= fraction <= 1.0:
        raise ValueError("fraction must be in [0, 1]")
    flat = np.asarray(spectrum, dtype=np.float64).reshape(-1)
    order = np.argsort(-np.abs(flat), kind="stable")
    sq = flat[order] ** 2
    cum = np.cumsum(sq)
    total = cum[-1] if cum.size else 0.0
    if fraction == 0.0 or total == 0.0:
        kept = 0
    else:
        kept = int(np.searchsorted(cum, fraction * total, side="left")) + 1
        kept = min(kept, int(np.count_nonzero(flat)))
    return _make_spectrum(flat, order, kept)


def energy_select_margin(spectrum, fraction: float) -> float:
    """Near-tie audit for compress_energy: relative distance between
    fraction*total and the two cumulative sums that bracket the cut. A value
    below ~1e-12 means a different (but equally valid) summation order could
    move the cut by one entry."""
    flat = np.asarray(spectrum, dtype=np.float64).reshape(-1)
    order = np.argsort(-np.abs(flat), kind="stable")
    cum = np.cumsum(flat[order] ** 2)
    if not cum.size or cum[-1] == 0.0:
        return np.inf
    target = fraction * cum[-1]
    pos = int(np.searchsorted(cum, target, side="left"))
    cand = [abs(cum[pos] - target)] if pos < cum.size else []
    if pos > 0:
        cand.append(abs(target - cum[pos - 1]))
    return min(cand) / cum[-1] if cand else np.inf


# ---------------------------------------------------------------------------
# dipole — dipole.py:85-152
# ---------------------------------------------------------------------------

def fdr(eta):  # dipole.py:85-89
    return -1.440 / (eta * eta) + 0.710 / eta + 0.668 + 0.0636 * eta


@dataclass(frozen=True)
class Dipole:
    sigma_t_prime: float
    alpha_prime: float
    sigma_tr: float
    z_r: float
    z_v: float


def derive_dipole_raw(sp, sa, eta) -> Dipole:  # dipole.py:100-116
    st = sp + sa
    ap = sp / st
    f = fdr(eta)
    a_boundary = (1.0 + f) / (1.0 - f)
    z_r = 1.0 / st
    return Dipole(st, ap, float(np.sqrt(3.0 * sa * st)), z_r,
                  z_r * (1.0 + 4.0 * a_boundary / 3.0))


def eval_rd(d: Dipole, r):  # dipole.py:119-132
    r = np.asarray(r, dtype=np.float64)
    d_r = np.sqrt(r * r + d.z_r * d.z_r)
    d_v = np.sqrt(r * r + d.z_v * d.z_v)
    s = d.sigma_tr
    term_r = d.z_r * (s + 1.0 / d_r) * np.exp(-s * d_r) / (d_r * d_r)
    term_v = d.z_v * (s + 1.0 / d_v) * np.exp(-s * d_v) / (d_v * d_v)
    return d.alpha_prime / (4.0 * np.pi) * (term_r + term_v)


def fresnel_transmittance(eta, cos_theta):  # dipole.py:135-152
    ci = np.clip(np.asarray(cos_theta, dtype=np.float64), 0.0, 1.0)
    if eta == 1.0:
        return np.ones_like(ci)
    sin2_t = (1.0 - ci * ci) / (eta * eta)
    tir = sin2_t >= 1.0
    ct = np.sqrt(np.maximum(1.0 - sin2_t, 0.0))
    rs = (ci - eta * ct) / (ci + eta * ct + 1e-300)
    rp = (eta * ci - ct) / (eta * ci + ct + 1e-300)
    ft = 1.0 - 0.5 * (rs * rs + rp * rp)
    return np.where(tir, 0.0, np.clip(ft, 0.0, 1.0))


# ---------------------------------------------------------------------------
# PCA basis — basisgen.py:90-191
# ---------------------------------------------------------------------------

def trapezoid_weights(nodes):  # basisgen.py:90-95
    w = np.empty_like(nodes)
    w[0] = (nodes[1] - nodes[0]) / 2.0
    w[-1] = (nodes[-1] - nodes[-2]) / 2.0
    w[1:-1] = (nodes[2:] - nodes[:-2]) / 2.0
    return w


def find_r_max(d: Dipole, ratio=1e-9):  # basisgen.py:98-112
    rd0 = float(eval_rd(d, 0.0))
    lo, hi = 0.0, 1.0
    while float(eval_rd(d, hi)) >= ratio * rd0:
        hi *= 2.0
    for _ in range(128):
        mid = 0.5 * (lo + hi)
        if float(eval_rd(d, mid)) < ratio * rd0:
            hi = mid
        else:
            lo = mid
    return hi


def r_nodes_for_box(sigma_box, eta, n_r=512):  # basisgen.py:115-129
    corner = derive_dipole_raw(sigma_box[0], sigma_box[2], eta)
    r_max = find_r_max(corner)
    return np.concatenate([[0.0], np.geomspace(1e-3, r_max, n_r - 1)])


def sigma_lattice(sigma_box, n_sp, n_sa):
    """Training materials: an n_sp x n_sa log-log lattice (basisgen.py:125-127
    uses lattice x lattice; BASELINE's 16/32/64 materials need 4x4, 8x4, 8x8 —
    SURVEY Appendix A)."""
    sp = np.geomspace(sigma_box[0], sigma_box[1], n_sp)
    sa = np.geomspace(sigma_box[2], sigma_box[3], n_sa)
    return np.stack(np.meshgrid(sp, sa, indexing="ij"), axis=-1).reshape(-1, 2)


def assemble_matrix(r_nodes, sigma_nodes, eta):  # basisgen.py:137-142
    sqrt_w = np.sqrt(trapezoid_weights(r_nodes))
    rows = np.empty((sigma_nodes.shape[0], r_nodes.shape[0]))
    for i, (sp, sa) in enumerate(sigma_nodes):
        rows[i] = eval_rd(derive_dipole_raw(sp, sa, eta), r_nodes) * sqrt_w
    return rows


def decompose(values, r_nodes, K):  # basisgen.py:145-169
    """Returns (bases (K, Nr) unweighted, singular values, U (M, K))."""
    u, s, vh = np.linalg.svd(values, full_matrices=False)
    weighted = vh[:K].copy()
    flip = np.ones(K)
    for i, row in enumerate(weighted):
        nz = np.flatnonzero(np.abs(row) > 1e-12 * np.abs(row).max())
        if nz.size and row[nz[0]] < 0.0:
            row *= -1.0
            flip[i] = -1.0
    return weighted / np.sqrt(trapezoid_weights(r_nodes)), s, u[:, :K] * flip


def project_row(bases, r_nodes, sp, sa, eta):  # basisgen.py:172-176
    w = trapezoid_weights(r_nodes)
    rd = eval_rd(derive_dipole_raw(sp, sa, eta), r_nodes)
    return (bases * w) @ rd


def project_material(bases, r_nodes, sigma_s_prime, sigma_a, eta):
    """basisgen.py:178-191 -> s (3, K)."""
    return np.stack([project_row(bases, r_nodes, float(sigma_s_prime[c]),
                                 float(sigma_a[c]), eta) for c in range(3)])


def basis_slopes(bases, r_nodes):  # transfer.py:155-156
    return (bases[:, 1:] - bases[:, :-1]) / np.diff(r_nodes)


# ---------------------------------------------------------------------------
# scattering-transfer rows — _kernels_np.py:142-158 (lerp mode) and the
# exact per-pair projection (SURVEY §8c "Exact per-pair projection")
# ---------------------------------------------------------------------------

def transfer_block(block_pos, positions, areas, r_nodes, bases, slopes):
    """(B, K, N): out[b,k,i] = (bases[k,j] + slopes[k,j]*(d - r_j)) * A_i."""
    nr = r_nodes.shape[0]
    diff = block_pos[:, None, :] - positions[None, :, :]
    d2 = (diff[..., 0] * diff[..., 0] + diff[..., 1] * diff[..., 1]) + diff[..., 2] * diff[..., 2]
    d = np.sqrt(d2)
    j = np.searchsorted(r_nodes, d, side="right") - 1
    np.clip(j, 0, nr - 2, out=j)
    frac = d - r_nodes[j]
    inside = d <= r_nodes[nr - 1]
    out = (bases[:, j] + slopes[:, j] * frac) * (areas * inside)
    return np.ascontiguousarray(out.swapaxes(0, 1))


def exact_projection_coeffs(U, singular_values, r_nodes, K):
    """P (K, M) with b_k(r) = sum_m P[k,m] R_d(r; sigma_m) on the nodes.

    decompose (basisgen.py:151-169) keeps V^T and discards U; since
    M = U S V^T with rows sqrt(w) R_d, V^T[k] = U[:,k]^T M / S_k, i.e. the
    unweighted basis b_k(r) = sum_m U[m,k]/S_k R_d(r; sigma_m).
    """
    return (U[:, :K] / singular_values[None, :K]).T.copy()


def transfer_block_exact(block_pos, positions, areas, r_max, sigma_nodes, eta, P):
    """(B, K, N) exact mode: b_k(d) = sum_m P[k,m] R_d(d; sigma_m), masked
    d <= r_max, times A_i (what the lerp in transfer_block approximates)."""
    diff = block_pos[:, None, :] - positions[None, :, :]
    d = np.sqrt((diff[..., 0] ** 2 + diff[..., 1] ** 2) + diff[..., 2] ** 2)
    rd = np.stack([eval_rd(derive_dipole_raw(sp, sa, eta), d)
                   for sp, sa in sigma_nodes])  # (M, B, N)
    out = np.einsum("km,mbn->bkn", P, rd)
    return out * (areas * (d <= r_max))[:, None, :]


# ---------------------------------------------------------------------------
# two-step compression — transfer.py:185-361, restated for a geometry image
# (identity atlas: part_count = 1, cell_of = arange) with the
# w0 / w1 transforms parameterised: (levels=full, w1="cdf97") is the
# reference exactly; (levels=L, w1="haar") is BASELINE's restatement.
# ---------------------------------------------------------------------------

TRANSFER_BLOCK = 64  # transfer.py:36


@dataclass
class Operator:
    cols: np.ndarray  # uint32 sorted w0 ids
    colptr: np.ndarray  # int64
    rowidx: np.ndarray  # uint32 w1 ids
    vals: np.ndarray  # float64
    kept_energy: float
    total_energy: float
    step1_entries: int

    @property
    def nnz(self):
        return int(self.rowidx.size)


def row_spectra_blocks(positions, areas, side, r_nodes, bases, levels, rows=None):
    """Yield (ids, (B, K, N) w0 spectra) — transfer.py:201-213."""
    n = positions.shape[0]
    slopes = basis_slopes(bases, r_nodes)
    ids_all = np.arange(n) if rows is None else np.asarray(rows)
    for lo in range(0, ids_all.size, TRANSFER_BLOCK):
        ids = ids_all[lo:lo + TRANSFER_BLOCK]
        block = transfer_block(positions[ids], positions, areas, r_nodes, bases, slopes)
        nb, K = len(ids), bases.shape[0]
        coeffs = haar2d_fwd(block.reshape(nb * K, side, side), levels)
        yield ids, coeffs.reshape(nb, K, n)


def step1(positions, areas, side, r_nodes, bases, keep, levels):
    """run_step1 + step1_unions (transfer.py:216-246) without the spill file.

    Returns (n, masks (K, N) bool, step1_entries per k, per-row sets dict
    when requested)."""
    n_dom = side * side
    n = max(int(round(keep * n_dom)), 1)
    K = bases.shape[0]
    masks = np.zeros((K, n_dom), bool)
    entries = [0] * K
    for ids, coeffs in row_spectra_blocks(positions, areas, side, r_nodes, bases, levels):
        for b in range(len(ids)):
            for k in range(K):
                spec = compress_top_n(coeffs[b, k], n)
                masks[k, spec.indices.astype(np.int64)] = True
                entries[k] += spec.count
    return n, masks, entries


def step2(positions, areas, side, r_nodes, bases, masks, entries, fraction,
          levels, w1="haar"):
    """compress_step2 + _threshold_columns (transfer.py:249-333)."""
    n_dom = side * side
    K = bases.shape[0]
    col_ids = [np.flatnonzero(masks[k]).astype(np.int64) for k in range(K)]
    columns = [np.zeros((c.size, n_dom), np.float32) for c in col_ids]
    for ids, coeffs in row_spectra_blocks(positions, areas, side, r_nodes, bases, levels):
        for k in range(K):
            columns[k][:, ids] = coeffs[:, k, col_ids[k]].T
    ops = []
    for k in range(K):
        ops.append(threshold_columns(columns[k], col_ids[k], side, fraction,
                                     entries[k], levels, w1))
    return ops


def threshold_columns(column_values, cols, side, fraction, step1_entries,
                      levels, w1="haar"):  # transfer.py:303-333
    n_dom = side * side
    specs = []
    for c0 in range(0, cols.size, 256):
        c1 = min(c0 + 256, cols.size)
        batch = column_values[c0:c1].astype(np.float64).reshape(-1, side, side)
        spectral = w_fwd(w1, batch, levels).reshape(c1 - c0, n_dom)
        for ci in range(c1 - c0):
            specs.append(compress_energy(spectral[ci], fraction))
    colptr = np.zeros(cols.size + 1, np.int64)
    for ci, sp in enumerate(specs):
        colptr[ci + 1] = colptr[ci] + sp.count
    rowidx = np.concatenate([s.indices for s in specs]) if specs else np.empty(0, np.uint32)
    vals = np.concatenate([s.values for s in specs]) if specs else np.empty(0)
    return Operator(cols.astype(np.uint32), colptr, rowidx.astype(np.uint32),
                    vals.astype(np.float64),
                    float(sum(s.kept_energy for s in specs)),
                    float(sum(s.total_energy for s in specs)), step1_entries)


def precompute_compressed(positions, areas, side, r_nodes, bases, step1_keep,
                          step2_fraction, levels=None, w1="haar"):
    """precompute_compressed (transfer.py:350-361) on a geometry image."""
    _, masks, entries = step1(positions, areas, side, r_nodes, bases, step1_keep, levels)
    return step2(positions, areas, side, r_nodes, bases, masks, entries,
                 step2_fraction, levels, w1)


def round_trip_f32(op: Operator) -> Operator:
    """PRTS1 stores vals as f32 (container.py:88, 103); the parity reference
    runs on the same rounded values."""
    return Operator(op.cols, op.colptr, op.rowidx,
                    op.vals.astype(np.float32).astype(np.float64),
                    op.kept_energy, op.total_energy, op.step1_entries)


# ---------------------------------------------------------------------------
# sparse apply — _kernels_np.py:239-257 / _kernels_nb.py:301-313
# ---------------------------------------------------------------------------

def csc_apply(cols, colptr, rowidx, vals, x_idx, x_val, out_len):
    """Serial reference order (_kernels_nb.py:301-313)."""
    out = np.zeros(out_len, np.float64)
    pos = np.searchsorted(cols, x_idx)
    ok = pos < cols.shape[0]
    ok &= cols[np.minimum(pos, cols.shape[0] - 1)] == x_idx
    pos = pos[ok]
    xv = np.asarray(x_val, np.float64)[ok]
    if pos.size == 0:
        return out
    starts = colptr[pos].astype(np.int64)
    counts = (colptr[pos + 1] - colptr[pos]).astype(np.int64)
    total = int(counts.sum())
    if total == 0:
        return out
    offs = np.repeat(np.cumsum(counts) - counts, counts)
    sel = np.arange(total, dtype=np.int64) - offs + np.repeat(starts, counts)
    # bincount accumulates sequentially in input order == the serial loop
    out += np.bincount(rowidx[sel].astype(np.int64),
                       weights=vals[sel] * np.repeat(xv, counts), minlength=out_len)
    return out


# ---------------------------------------------------------------------------
# light projection (a) — lighting.py:293-336, envmap.py:45-66
# ---------------------------------------------------------------------------

def face_directions(side):  # envmap.py:45-58
    t = (np.arange(side) + 0.5) / side * 2.0 - 1.0
    v, u = np.meshgrid(t, t, indexing="ij")
    one = np.ones_like(u)
    raw = np.stack([
        np.stack([one, -v, -u], axis=-1),
        np.stack([-one, -v, u], axis=-1),
        np.stack([u, one, v], axis=-1),
        np.stack([u, -one, -v], axis=-1),
        np.stack([u, -v, one], axis=-1),
        np.stack([-u, -v, -one], axis=-1),
    ])
    return raw / np.linalg.norm(raw, axis=-1, keepdims=True)


def face_solid_angles(side):  # envmap.py:61-66
    t = (np.arange(side) + 0.5) / side * 2.0 - 1.0
    v, u = np.meshgrid(t, t, indexing="ij")
    w = 4.0 / (side * side) / np.power(u * u + v * v + 1.0, 1.5)
    return np.tile(w, (6, 1, 1))


def visibility_weights(normals, side, eta=1.0, visibility=None):
    """lighting.py:318-329: W = V * F_t(eta, cos+) * cos+ * d_omega.

    BASELINE's light transfer is unshadowed (V = 1) with eta_light = 1
    (F_t == 1, dipole.py:142-144) — SURVEY Appendix A."""
    dirs = face_directions(side).reshape(-1, 3)
    dom = face_solid_angles(side).reshape(-1)
    cosp = np.clip(normals @ dirs.T, 0.0, 1.0)
    vis = 1.0 if visibility is None else visibility
    return vis * fresnel_transmittance(eta, cosp) * cosp * dom[None, :]


def env_transfer_w2(normals, side):
    """W in the w2 (per-face full Haar) domain, as fold_visibility builds it
    (transfer.py:407-411), stored as float32 (BASELINE: fp32 transfer)."""
    w = visibility_weights(normals, side)
    n = normals.shape[0]
    w2 = haar2d_fwd(w.reshape(n * 6, side, side)).reshape(n, 6 * side * side)
    return w2.astype(np.float32)


def project_environment(faces, n_keep=128):
    """lighting.py:293-305: faces (6, s, s, 3) -> 3 Spectrum (top n_keep)."""
    out = []
    for c in range(3):
        coeffs = haar2d_fwd(np.ascontiguousarray(faces[..., c], dtype=np.float64))
        out.append(compress_top_n(coeffs.reshape(-1), n_keep))
    return out


def env_irradiance(w2_t32, spectra):
    """E[:, c] = sum over the (sorted) union of the three channels' kept w2
    ids of W^{w2}[:, l] * L_c[l] (L_c[l] = 0 where channel c dropped l);
    fp64 accumulate in ascending l order. Equals
    ambient_irradiance_dense(W, reconstruct_environment(spectra)) by Parseval
    (lighting.py:308-336)."""
    n = w2_t32.shape[0]
    union = np.unique(np.concatenate([s.indices for s in spectra])).astype(np.int64)
    lc = np.zeros((3, union.size))
    for c in range(3):
        pos = np.searchsorted(union, spectra[c].indices.astype(np.int64))
        lc[c, pos] = spectra[c].values
    E = np.zeros((n, 3))
    for q, l in enumerate(union):
        col = w2_t32[:, l].astype(np.float64)
        for c in range(3):
            if lc[c, q] != 0.0:
                E[:, c] = E[:, c] + col * lc[c, q]
    return E


def sh_irradiance(T32, Lsh):
    """E[:, c] = sum_l T[:, l] * L[l, c], fp64 accumulate in l order
    (the SH analogue of ambient_irradiance_dense, lighting.py:332-336)."""
    E = np.zeros((T32.shape[0], 3))
    for l in range(T32.shape[1]):
        col = T32[:, l].astype(np.float64)
        for c in range(3):
            E[:, c] = E[:, c] + col * float(Lsh[l, c])
    return E


# ---------------------------------------------------------------------------
# the frame — runtime.py:109-216 (Scene.relight / set_material / _finish)
# ---------------------------------------------------------------------------

def select_irradiance(E, side, levels, e_keep):
    """_stage1_irradiance (runtime.py:109-118): per channel w0 Haar, top-n."""
    n_dom = side * side
    keep = max(1, int(round(e_keep * n_dom)))
    spectra = []
    for c in range(3):
        coeffs = haar2d_fwd(E[:, c].reshape(1, side, side), levels).reshape(-1)
        spectra.append(compress_top_n(coeffs, keep))
    return spectra


def transfer_stage(ops, spectra, n_dom):
    """_stage2_transfer (runtime.py:138-150) -> vk (K, 3, n_dom)."""
    vk = np.zeros((len(ops), 3, n_dom))
    for k, op in enumerate(ops):
        for c in range(3):
            vk[k, c] = csc_apply(op.cols, op.colptr, op.rowidx, op.vals,
                                 spectra[c].indices, spectra[c].values, n_dom)
    return vk


def finish(vk, weights, side, levels, w1, normals, positions, cam_pos, eta):
    """_finish + _stage5_reconstruct + _shade (runtime.py:155-168, 202-216)."""
    summed = np.einsum("ck,kcd->cd", weights, vk)
    scatter = np.empty((side * side, 3))
    for c in range(3):
        scatter[:, c] = w_inv(w1, summed[c].reshape(1, side, side), levels).reshape(-1)
    view = cam_pos[None, :] - positions
    view = view / np.linalg.norm(view, axis=1, keepdims=True)
    cos = np.clip(np.einsum("ij,ij->i", normals, view), 0.0, 1.0)
    ft = fresnel_transmittance(eta, cos)
    unclamped = scatter * (ft / np.pi)[:, None]
    return np.maximum(unclamped, 0.0), unclamped, scatter


def relight(E, ops, bases, r_nodes, material, side, levels, w1, e_keep,
            normals, positions, cam_pos):
    """Full frame: returns dict(radiance, radiance_unclamped, scatter, vk,
    spectra, weights)."""
    sp, sa, eta = material
    spectra = select_irradiance(E, side, levels, e_keep)
    vk = transfer_stage(ops, spectra, side * side)
    weights = project_material(bases, r_nodes, sp, sa, eta)
    rad, unc, scatter = finish(vk, weights, side, levels, w1, normals, positions,
                               cam_pos, eta)
    return dict(radiance=rad, radiance_unclamped=unc, scatter=scatter, vk=vk,
                spectra=spectra, weights=weights)


def parity_error(got, ref, tau=1e-3):
    """max_i |got-ref| / max(|ref_i|, tau * max|ref|)."""
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    floor = tau * np.abs(ref).max()
    if floor == 0.0:
        return float(np.abs(got).max())
    return float((np.abs(got - ref) / np.maximum(np.abs(ref), floor)).max())


def coeff_tile(r, c, side, levels):
    """Spatial 2^L x 2^L tile that coefficient (r, c) of an L-level Mallat
    layout belongs to (the L-level transform is tile-local)."""
    for lvl in range(1, levels + 1):
        half = side >> lvl
        if r >= half or c >= half:
            sh = levels - lvl
            return ((r % half) >> sh, (c % half) >> sh)
    return (r, c)


def env_transfer_w2_exact(normals32, side):
    """env_transfer_w2 with the dot product written out in the device's
    order ((n0 d0 + n1 d1) + n2 d2) so the float32 table is bitwise
    reproducible (BLAS may fuse or reorder `normals @ dirs.T`)."""
    n = np.asarray(normals32, np.float64)
    dirs = face_directions(side).reshape(-1, 3)
    dom = face_solid_angles(side).reshape(-1)
    cos = (n[:, 0:1] * dirs[None, :, 0] + n[:, 1:2] * dirs[None, :, 1]) + n[:, 2:3] * dirs[None, :, 2]
    w = np.clip(cos, 0.0, 1.0) * dom[None, :]
    w2 = haar2d_fwd(w.reshape(n.shape[0] * 6, side, side)).reshape(n.shape[0], 6 * side * side)
    return w2.astype(np.float32)


def csr_rows_apply(rowptr, cols, vals, rows, x):
    """CPU port of the transfer apply for a subset of operator rows stored in
    the device's tile-major CSR layout: out[q, c] = sum_p vals[p] x[c, cols[p]]
    over row rows[q] (the same products csc_apply accumulates column by
    column, _kernels_nb.py:301-313). x: (3, N) masked E spectrum."""
    rows = np.asarray(rows, np.int64)
    starts = rowptr[rows].astype(np.int64)
    counts = (rowptr[rows + 1] - rowptr[rows]).astype(np.int64)
    total = int(counts.sum())
    out = np.zeros((rows.size, x.shape[0]))
    if total == 0:
        return out
    offs = np.repeat(np.cumsum(counts) - counts, counts)
    sel = np.arange(total, dtype=np.int64) - offs + np.repeat(starts, counts)
    seg = np.repeat(np.arange(rows.size), counts)
    c = cols[sel].astype(np.int64)
    v = vals[sel].astype(np.float64)
    for ch in range(x.shape[0]):
        out[:, ch] = np.bincount(seg, weights=v * x[ch, c], minlength=rows.size)
    return out


# ---------------------------------------------------------------------------
# Direct lights with shadow rays: lighting.py:101-290,
# _kernels_nb.py:208-298 / _kernels_np.py:165-232. The geometry image's grid
# triangulation is the mesh the shadow rays see.
# ---------------------------------------------------------------------------
RAY_OFFSET_SCALE = 1e-4       # lighting.py:23 (of the bbox diagonal)
SPHERE_LIGHT_SAMPLES = 64     # lighting.py:24 (8 x 8 midpoint cone strata)


def grid_triangles(side):
    """Two triangles per geometry-image cell: (i00, i01, i11), (i00, i11, i10)."""
    r, c = np.meshgrid(np.arange(side - 1), np.arange(side - 1), indexing="ij")
    i00 = (r * side + c).reshape(-1)
    i01, i10 = i00 + 1, i00 + side
    i11 = i10 + 1
    t = np.empty((i00.size * 2, 3), np.int32)
    t[0::2] = np.stack([i00, i01, i11], 1)
    t[1::2] = np.stack([i00, i11, i10], 1)
    return t


def tri_any_hit(o, d, tmax, v0, e1, e2):  # _kernels_np.py:165-176 (row-aligned batches)
    pv = np.cross(d, e2)
    det = np.einsum("ij,ij->i", e1, pv)
    ok = np.abs(det) > 1e-14
    inv = np.where(ok, 1.0 / np.where(ok, det, 1.0), 0.0)
    tv = o - v0
    u = np.einsum("ij,ij->i", tv, pv) * inv
    qv = np.cross(tv, e1)
    v = np.einsum("ij,ij->i", d, qv) * inv
    t = np.einsum("ij,ij->i", e2, qv) * inv
    return ok & (u >= 0.0) & (u <= 1.0) & (v >= 0.0) & (u + v <= 1.0) & (t > 1e-9) & (t < tmax)


def any_hit(origins, dirs, tmax, vertices, tris, chunk=1 << 22):
    """Brute force over every triangle (the checker; any-hit is independent
    of the acceleration structure)."""
    v = np.asarray(vertices, np.float64)
    v0 = v[tris[:, 0]]
    e1 = v[tris[:, 1]] - v0
    e2 = v[tris[:, 2]] - v0
    nt = v0.shape[0]
    out = np.zeros(origins.shape[0], bool)
    per = max(1, chunk // nt)
    for a in range(0, origins.shape[0], per):
        b = min(a + per, origins.shape[0])
        m = b - a
        o = np.repeat(origins[a:b], nt, axis=0)
        d = np.repeat(dirs[a:b], nt, axis=0)
        tm = np.repeat(tmax[a:b], nt)
        h = tri_any_hit(o, d, tm, np.tile(v0, (m, 1)), np.tile(e1, (m, 1)), np.tile(e2, (m, 1)))
        out[a:b] = h.reshape(m, nt).any(axis=1)
    return out


def _cone_strata():  # lighting.py:191-195
    side = int(np.sqrt(SPHERE_LIGHT_SAMPLES))
    u = (np.arange(side) + 0.5) / side
    u1, u2 = np.meshgrid(u, u, indexing="ij")
    return u1.ravel(), u2.ravel()


def _orthonormal_frame(axis):  # lighting.py:200-205
    helper = np.where(np.abs(axis[..., 2:3]) < 0.9, [0.0, 0.0, 1.0], [1.0, 0.0, 0.0])
    t1 = np.cross(axis, helper)
    t1 /= np.linalg.norm(t1, axis=-1, keepdims=True)
    t2 = np.cross(axis, t1)
    return t1, t2


def irradiance_direct(positions, normals, lights, vertices, tris, eta):
    """lighting.py:208-249 (+ _sphere_light_irradiance :252-290). lights: list
    of ("point", position, intensity) / ("directional", direction (unit,
    light -> scene), irradiance) / ("sphere", center, radius, radiance)."""
    pos = np.asarray(positions, np.float64)
    nrm = np.asarray(normals, np.float64)
    n = pos.shape[0]
    v = np.asarray(vertices, np.float64)
    bbox_diag = float(np.linalg.norm(v.max(axis=0) - v.min(axis=0)))
    origins = pos + RAY_OFFSET_SCALE * bbox_diag * nrm
    e_out = np.zeros((n, 3))
    for light in lights:
        kind = light[0]
        if kind == "point":
            _, lp, inten = light
            dvec = np.asarray(lp, np.float64)[None, :] - pos
            dist = np.linalg.norm(dvec, axis=1)
            wi = dvec / dist[:, None]
            cos = np.einsum("ij,ij->i", nrm, wi)
            lit = cos > 0.0
            vis = np.zeros(n, bool)
            if lit.any():
                vis[lit] = ~any_hit(origins[lit], wi[lit], dist[lit], v, tris)
            weight = np.where(lit & vis, fresnel_transmittance(eta, np.clip(cos, 0.0, 1.0))
                              * np.clip(cos, 0.0, 1.0) / (dist * dist), 0.0)
            e_out += weight[:, None] * np.asarray(inten, np.float64)[None, :]
        elif kind == "directional":
            _, direction, irr = light
            wi = -np.asarray(direction, np.float64)
            cos = nrm @ wi
            lit = cos > 0.0
            vis = np.zeros(n, bool)
            if lit.any():
                far = np.full(int(lit.sum()), 4.0 * bbox_diag + 1.0)
                vis[lit] = ~any_hit(origins[lit], np.tile(wi, (int(lit.sum()), 1)), far, v, tris)
            weight = np.where(lit & vis, fresnel_transmittance(eta, np.clip(cos, 0.0, 1.0))
                              * np.clip(cos, 0.0, 1.0), 0.0)
            e_out += weight[:, None] * np.asarray(irr, np.float64)[None, :]
        elif kind == "sphere":
            _, center, radius, rad = light
            axis = np.asarray(center, np.float64)[None, :] - pos
            dist = np.linalg.norm(axis, axis=1)
            if np.any(dist <= radius):
                raise ValueError("sphere light overlaps the surface")
            axis = axis / dist[:, None]
            sin_max = radius / dist
            cos_max = np.sqrt(np.clip(1.0 - sin_max * sin_max, 0.0, 1.0))
            omega = 2.0 * np.pi * (1.0 - cos_max)
            u1, u2 = _cone_strata()
            t1, t2 = _orthonormal_frame(axis)
            ct = 1.0 - u1[None, :] * (1.0 - cos_max[:, None])
            st = np.sqrt(np.clip(1.0 - ct * ct, 0.0, 1.0))
            phi = 2.0 * np.pi * u2[None, :]
            dirs = (axis[:, None, :] * ct[..., None]
                    + t1[:, None, :] * (st * np.cos(phi))[..., None]
                    + t2[:, None, :] * (st * np.sin(phi))[..., None])
            cos = np.einsum("ij,isj->is", nrm, dirs)
            lit = cos > 0.0
            proj = dist[:, None] * ct
            under = proj * proj - (dist * dist - radius * radius)[:, None]
            t_hit = proj - np.sqrt(np.clip(under, 0.0, None))
            vis = np.zeros_like(lit)
            if lit.any():
                ray_o = np.repeat(origins, len(u1), axis=0)[lit.ravel()]
                vis[lit] = ~any_hit(ray_o, dirs[lit], t_hit[lit], v, tris)
            weight = np.where(lit & vis, fresnel_transmittance(eta, np.clip(cos, 0.0, 1.0))
                              * np.clip(cos, 0.0, 1.0), 0.0).mean(axis=1) * omega
            e_out += weight[:, None] * np.asarray(rad, np.float64)[None, :]
        else:
            raise TypeError(f"unsupported light {kind}")
    return e_out


# ---------------------------------------------------------------------------
# visibility precompute and ambient folding —
# transfer.py:368-451, lighting.py:318-329
# ---------------------------------------------------------------------------

FOLD_FRACTION = 0.9999  # transfer.py:35 DEFAULT_FOLD_FRACTION
ENV_COEFF_KEEP = 128    # runtime.py:34


def precompute_visibility(positions, normals, vertices, tris, face_side=16):
    """precompute_visibility (transfer.py:368-391): binary upper-hemisphere
    visibility (N, 6 s^2) over the cubemap texel directions; rays from
    p + offset n toward every direction with n.d > 0, any hit within
    4 diag + 1 occludes. Brute-force any-hit (the answer is independent of
    the acceleration structure)."""
    v = np.asarray(vertices, np.float64)
    diag = float(np.linalg.norm(v.max(axis=0) - v.min(axis=0)))
    ray_offset = RAY_OFFSET_SCALE * diag
    dirs = face_directions(face_side).reshape(-1, 3)
    n, d = positions.shape[0], dirs.shape[0]
    origins = positions + ray_offset * normals
    cos = normals @ dirs.T
    far = 4.0 * diag + 1.0
    vis = np.zeros((n, d))
    si, di = np.nonzero(cos > 0.0)
    if si.size:
        hits = any_hit(origins[si], dirs[di], np.full(si.size, far), v, tris)
        vis[si, di] = ~hits
    return vis


def fold_visibility(ops, vis, normals, side, face_side, eta, fraction=FOLD_FRACTION,
                    levels=None):
    """fold_visibility (transfer.py:394-451) for an identity atlas: per k the
    operator (w1 rows x kept w0 columns) times v~ = w0(w2(W)) restricted to
    its columns, then compress_energy per direction column. W =
    visibility_weights with the material eta; w2 = per-face full Haar over
    the direction axis; w0 = the L-level (None = full) Haar over samples.
    Returns the folded operators and the dense (w1, D) products per k."""
    n = normals.shape[0]
    d = 6 * face_side * face_side
    w = visibility_weights(normals, face_side, eta, vis)
    w2 = haar2d_fwd(np.ascontiguousarray(w.reshape(n * 6, face_side, face_side))).reshape(n, d)
    v_tilde = haar2d_fwd(np.ascontiguousarray(w2.T.reshape(d, side, side)), levels)
    v_tilde = v_tilde.reshape(d, n).T
    out, dense_folded = [], []
    for op in ops:
        cols = op.cols.astype(np.int64)
        dense = np.zeros((n, cols.size))
        for ci in range(cols.size):
            sl = slice(op.colptr[ci], op.colptr[ci + 1])
            dense[op.rowidx[sl].astype(np.int64), ci] = op.vals[sl]
        folded = dense @ v_tilde[cols, :]
        dense_folded.append(folded)
        specs = [compress_energy(folded[:, e], fraction) for e in range(d)]
        fcols = np.flatnonzero([s.count for s in specs]).astype(np.uint32)
        keep = [specs[int(c)] for c in fcols]
        colptr = np.zeros(fcols.size + 1, np.int64)
        for ci, sp in enumerate(keep):
            colptr[ci + 1] = colptr[ci] + sp.count
        out.append(Operator(
            fcols, colptr,
            np.concatenate([s.indices for s in keep]).astype(np.uint32) if keep
            else np.empty(0, np.uint32),
            np.concatenate([s.values for s in keep]) if keep else np.empty(0),
            float(sum(s.kept_energy for s in specs)), float(sum(s.total_energy for s in specs)),
            int(np.count_nonzero(folded))))
    return out, dense_folded


def ambient_vk(folded_ops, spectra, n_dom):
    """The folded ambient term of _stage2_transfer (runtime.py:146-149):
    vk[k, c] = folded_k applied to the channel's w2 environment spectrum."""
    vk = np.zeros((len(folded_ops), 3, n_dom))
    for k, op in enumerate(folded_ops):
        for c in range(3):
            vk[k, c] = csc_apply(op.cols, op.colptr, op.rowidx, op.vals, spectra[c].indices,
                                 spectra[c].values, n_dom)
    return vk


# ---------------------------------------------------------------------------
# rasterisation: render_image / raster_fill
# ---------------------------------------------------------------------------
def camera_basis(position, look_at, up):
    """The camera frame of _project_vertices (runtime.py:248-256)."""
    position = np.asarray(position, np.float64)
    fwd = np.asarray(look_at, np.float64) - position
    fwd = fwd / np.linalg.norm(fwd)
    right = np.cross(fwd, np.asarray(up, np.float64))
    nr = np.linalg.norm(right)
    if nr < 1e-12:
        raise ValueError("camera up vector is parallel to the view direction")
    right /= nr
    upv = np.cross(right, fwd)
    return right, upv, fwd


def project_vertices(vertices, position, look_at, up, fov_y_degrees, width, height):
    """_project_vertices (runtime.py:247-273). The three camera-space dot
    products are written as left-to-right element sums (x·r0 + y·r1) + z·r2
    (the reference's `rel @ right` goes through BLAS; the GPU uses this same
    order, so this checker and the kernel agree bitwise)."""
    right, upv, fwd = camera_basis(position, look_at, up)
    rel = np.asarray(vertices, np.float64) - np.asarray(position, np.float64)

    def dot(a):
        return (rel[:, 0] * a[0] + rel[:, 1] * a[1]) + rel[:, 2] * a[2]

    x, y, z = dot(right), dot(upv), dot(fwd)
    near = 1e-3
    f = 1.0 / np.tan(np.radians(fov_y_degrees) / 2.0)
    aspect = width / height
    with np.errstate(divide="ignore", invalid="ignore"):
        ndc_x = (x * f / aspect) / z
        ndc_y = (y * f) / z
    sx = (ndc_x * 0.5 + 0.5) * width
    sy = (0.5 - ndc_y * 0.5) * height
    iw = np.where(z > near, 1.0 / z, 0.0)
    zn = np.where(z > near, z, np.inf)
    return sx, sy, zn, iw


def raster_fill(tris, sx, sy, zn, iw, colors, zbuf, img):
    """raster_fill (_kernels_np.py:264-313 / _kernels_nb.py:316-359): triangles
    in order, strict z-test, perspective-correct colour; zbuf/img in place."""
    height, width = zbuf.shape
    for t in range(tris.shape[0]):
        i0, i1, i2 = int(tris[t, 0]), int(tris[t, 1]), int(tris[t, 2])
        if iw[i0] <= 0.0 or iw[i1] <= 0.0 or iw[i2] <= 0.0:
            continue
        x0, y0, x1, y1, x2, y2 = sx[i0], sy[i0], sx[i1], sy[i1], sx[i2], sy[i2]
        area = (x1 - x0) * (y2 - y0) - (y1 - y0) * (x2 - x0)
        if area == 0.0:
            continue
        xmin = max(int(math.floor(min(x0, x1, x2))), 0)
        xmax = min(int(math.ceil(max(x0, x1, x2))), width - 1)
        ymin = max(int(math.floor(min(y0, y1, y2))), 0)
        ymax = min(int(math.ceil(max(y0, y1, y2))), height - 1)
        if xmin > xmax or ymin > ymax:
            continue
        pxg = (np.arange(xmin, xmax + 1, dtype=np.float64) + 0.5)[None, :]
        pyg = (np.arange(ymin, ymax + 1, dtype=np.float64) + 0.5)[:, None]
        w0 = (x2 - x1) * (pyg - y1) - (y2 - y1) * (pxg - x1)
        w1 = (x0 - x2) * (pyg - y2) - (y0 - y2) * (pxg - x2)
        w2 = (x1 - x0) * (pyg - y0) - (y1 - y0) * (pxg - x0)
        if area > 0.0:
            inside = (w0 >= 0.0) & (w1 >= 0.0) & (w2 >= 0.0)
        else:
            inside = (w0 <= 0.0) & (w1 <= 0.0) & (w2 <= 0.0)
        l0, l1, l2 = w0 / area, w1 / area, w2 / area
        z = l0 * zn[i0] + l1 * zn[i1] + l2 * zn[i2]
        sub_z = zbuf[ymin:ymax + 1, xmin:xmax + 1]
        upd = inside & (z < sub_z)
        if not upd.any():
            continue
        wi = l0 * iw[i0] + l1 * iw[i1] + l2 * iw[i2]
        sub_img = img[ymin:ymax + 1, xmin:xmax + 1]
        for c in range(3):
            num = (l0 * (colors[i0, c] * iw[i0]) + l1 * (colors[i1, c] * iw[i1])
                   + l2 * (colors[i2, c] * iw[i2]))
            with np.errstate(divide="ignore", invalid="ignore"):
                sub_img[..., c] = np.where(upd, num / wi, sub_img[..., c])
        sub_z[upd] = z[upd]
    return zbuf


def linear_to_srgb(x):  # envmap.py:74-76
    x = np.clip(np.asarray(x, np.float64), 0.0, 1.0)
    return np.where(x <= 0.0031308, x * 12.92, 1.055 * np.power(x, 1.0 / 2.4) - 0.055)


def encode_srgb8(x, exposure=1.0):
    """The 8-bit quantisation of render_image (runtime.py:245) and of the
    service frame payload (service.py:181)."""
    return (linear_to_srgb(np.asarray(x, np.float64) * exposure) * 255.0 + 0.5).astype(np.uint8)


def render_image(vertices, tris, source_vertex, radiance, position, look_at, up, fov_y_degrees,
                 width, height, exposure=1.0, background=(0.0, 0.0, 0.0)):
    """render_image (runtime.py:230-245): returns (u8 image, linear image, zbuf)."""
    if width < 1 or height < 1:
        raise ValueError("image dimensions must be positive")
    colors = np.zeros((np.asarray(vertices).shape[0], 3))
    colors[np.asarray(source_vertex)] = radiance
    sx, sy, zn, iw = project_vertices(vertices, position, look_at, up, fov_y_degrees, width, height)
    zbuf = np.full((height, width), np.inf)
    img = np.empty((height, width, 3))
    img[:] = np.asarray(background, np.float64)
    raster_fill(np.ascontiguousarray(tris, np.int64), sx, sy, zn, iw, colors, zbuf, img)
    return encode_srgb8(img, exposure), img, zbuf
