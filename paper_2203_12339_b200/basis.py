"""Dipole PCA basis (offline setup) and per-edit material weights (path c).

The basis itself — R_d sampled on a (sigma_s', sigma_a) lattice x 512 radial
nodes, SVD, sign fix — is an offline, sub-second LAPACK job the survey says
to ship as data rather than port; it is computed here
on the host with the reference's conventions (basisgen.py:90-169) and then
lives on the device. ``project_material`` (basisgen.py:178-191) is the
per-edit hot call and runs in CUDA (``sss_material_weights``).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .config import ETA, N_R, SIGMA_BOX

# ---------------------------------------------------------------------------
# data model (dipole.py:30-69, basisgen.py:56-87)
# ---------------------------------------------------------------------------


def _as_rgb(v, name):
    a = np.asarray(v, dtype=np.float64)
    if a.ndim == 0:
        a = np.repeat(a[None], 3)
    if a.shape != (3,):
        raise ValueError(f"{name} must be a scalar or length-3 per-channel array")
    return a


@dataclass(frozen=True)
class OpticalMaterial:
    """Editable translucent material (dipole.py:30-69)."""

    sigma_s_prime: np.ndarray
    sigma_a: np.ndarray
    g: float = 0.0
    eta: float = 1.3

    def __post_init__(self):
        object.__setattr__(self, "sigma_s_prime", _as_rgb(self.sigma_s_prime, "sigma_s_prime"))
        object.__setattr__(self, "sigma_a", _as_rgb(self.sigma_a, "sigma_a"))
        if not np.all(self.sigma_s_prime > 0.0) or not np.all(np.isfinite(self.sigma_s_prime)):
            raise ValueError("sigma_s_prime must be positive and finite per channel")
        if not np.all(self.sigma_a > 0.0) or not np.all(np.isfinite(self.sigma_a)):
            raise ValueError("sigma_a must be positive and finite per channel")
        if not -1.0 < self.g < 1.0:
            raise ValueError("g must lie in (-1, 1)")
        if not 1.0 <= self.eta <= 3.0:
            raise ValueError("eta must lie in [1.0, 3.0]")

    def channel(self, c: int):
        return float(self.sigma_s_prime[c]), float(self.sigma_a[c])


@dataclass(frozen=True)
class DiffusionBasis:
    """Top-K radial bases, quadrature-unweighted (basisgen.py:56-81), plus the
    left singular vectors the exact per-pair projection needs."""

    r_nodes: np.ndarray
    bases: np.ndarray  # (K, N_r)
    singular_values: np.ndarray
    sigma_nodes: np.ndarray  # (M, 2) training materials
    U: np.ndarray  # (M, K)
    eta: float = ETA
    g: float = 0.0
    sigma_box: tuple = SIGMA_BOX
    _dev: dict = field(default_factory=dict, repr=False, compare=False)

    @property
    def K(self) -> int:
        return int(self.bases.shape[0])

    @property
    def r_max(self) -> float:
        return float(self.r_nodes[-1])

    @property
    def r_weights(self) -> np.ndarray:
        return trapezoid_weights(self.r_nodes)

    def device(self, device="cuda"):
        """Device copies used by the kernels (cached)."""
        key = str(device)
        if key not in self._dev:
            bw = self.bases * self.r_weights  # (basis.bases * w), basisgen.py:176
            self._dev[key] = dict(
                bw=torch.as_tensor(bw, dtype=torch.float64, device=device).contiguous(),
                r_nodes=torch.as_tensor(self.r_nodes, dtype=torch.float64, device=device),
                bases=torch.as_tensor(self.bases, dtype=torch.float64, device=device).contiguous(),
            )
        return self._dev[key]


@dataclass(frozen=True)
class MaterialWeights:
    s: np.ndarray  # (3, K)
    material: OpticalMaterial = None


# ---------------------------------------------------------------------------
# offline basis construction (host)
# ---------------------------------------------------------------------------


def fdr(eta):
    return -1.440 / (eta * eta) + 0.710 / eta + 0.668 + 0.0636 * eta


def _derive(sp, sa, eta):
    st = sp + sa
    f = fdr(eta)
    a = (1.0 + f) / (1.0 - f)
    z_r = 1.0 / st
    return sp / st, math.sqrt(3.0 * sa * st), z_r, z_r * (1.0 + 4.0 * a / 3.0)


def eval_rd(sp, sa, eta, r):
    """R_d(r) (dipole.py:119-132), vectorised over r."""
    ap, s, z_r, z_v = _derive(sp, sa, eta)
    r = np.asarray(r, dtype=np.float64)
    d_r = np.sqrt(r * r + z_r * z_r)
    d_v = np.sqrt(r * r + z_v * z_v)
    term_r = z_r * (s + 1.0 / d_r) * np.exp(-s * d_r) / (d_r * d_r)
    term_v = z_v * (s + 1.0 / d_v) * np.exp(-s * d_v) / (d_v * d_v)
    return ap / (4.0 * np.pi) * (term_r + term_v)


def trapezoid_weights(nodes):
    w = np.empty_like(nodes)
    w[0] = (nodes[1] - nodes[0]) / 2.0
    w[-1] = (nodes[-1] - nodes[-2]) / 2.0
    w[1:-1] = (nodes[2:] - nodes[:-2]) / 2.0
    return w


def find_r_max(sp, sa, eta, ratio=1e-9):
    """Bisection to R_d(r)/R_d(0) < ratio (basisgen.py:98-112)."""
    rd0 = float(eval_rd(sp, sa, eta, 0.0))
    lo, hi = 0.0, 1.0
    while float(eval_rd(sp, sa, eta, hi)) >= ratio * rd0:
        hi *= 2.0
        if hi > 1e9:
            raise RuntimeError("R_d failed to decay")
    for _ in range(128):
        mid = 0.5 * (lo + hi)
        if float(eval_rd(sp, sa, eta, mid)) < ratio * rd0:
            hi = mid
        else:
            lo = mid
    return hi


def build_basis(K: int, lattice=(4, 4), sigma_box=SIGMA_BOX, eta=ETA, n_r=N_R) -> DiffusionBasis:
    """build_sample_grid + assemble_matrix + decompose (basisgen.py:115-169)
    with an n_sp x n_sa log-log training lattice."""
    sp_min, sp_max, sa_min, sa_max = sigma_box
    r_max = find_r_max(sp_min, sa_min, eta)
    r_nodes = np.concatenate([[0.0], np.geomspace(1e-3, r_max, n_r - 1)])
    sp = np.geomspace(sp_min, sp_max, lattice[0])
    sa = np.geomspace(sa_min, sa_max, lattice[1])
    nodes = np.stack(np.meshgrid(sp, sa, indexing="ij"), axis=-1).reshape(-1, 2)
    sqrt_w = np.sqrt(trapezoid_weights(r_nodes))
    M = np.stack([eval_rd(a, b, eta, r_nodes) * sqrt_w for a, b in nodes])
    if not 1 <= K <= min(M.shape):
        raise ValueError(f"K must lie in [1, {min(M.shape)}]")
    u, s, vh = np.linalg.svd(M, full_matrices=False)
    weighted = vh[:K].copy()
    flip = np.ones(K)
    for i, row in enumerate(weighted):
        nz = np.flatnonzero(np.abs(row) > 1e-12 * np.abs(row).max())
        if nz.size and row[nz[0]] < 0.0:
            row *= -1.0
            flip[i] = -1.0
    return DiffusionBasis(r_nodes=r_nodes, bases=weighted / sqrt_w, singular_values=s,
                          sigma_nodes=nodes, U=u[:, :K] * flip, eta=eta, sigma_box=sigma_box)


def basis_for(cfg) -> DiffusionBasis:
    return build_basis(cfg.K, cfg.lattice)


# ---------------------------------------------------------------------------
# per-edit material weights on the GPU (basisgen.py:178-191)
# ---------------------------------------------------------------------------


def material_weights_device(basis: DiffusionBasis, material: OpticalMaterial, out=None,
                            sigma_dev=None, stream=None):
    """s (3, K) fp64 on the device; sigma_dev: optional preallocated (7,)
    buffer {sp[3], sa[3], eta}."""
    dev = basis.device()
    if sigma_dev is None:
        sigma_dev = torch.tensor(np.concatenate([material.sigma_s_prime, material.sigma_a,
                                                 [material.eta]]),
                                 dtype=torch.float64, device="cuda")
    if out is None:
        out = torch.empty((3, basis.K), dtype=torch.float64, device="cuda")
    _lib.call("sss_material_weights", _lib.ptr(dev["bw"]), _lib.ptr(dev["r_nodes"]),
              basis.K, len(basis.r_nodes), _lib.ptr(sigma_dev), _lib.ptr(out),
              _lib.stream_ptr(stream))
    return out


def project_material(basis: DiffusionBasis, material: OpticalMaterial, channel=None):
    """Reference API (basisgen.py:178-191): returns MaterialWeights(s (3, K))
    or the (K,) row for one channel."""
    s = material_weights_device(basis, material).cpu().numpy()
    if channel is not None:
        return s[channel]
    return MaterialWeights(s=s, material=material)
