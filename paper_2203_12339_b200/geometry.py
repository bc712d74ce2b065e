"""Geometry images: the surface data model the hot path runs on.

BASELINE's scenes are S x S geometry images built by octahedral mapping of a
perturbed sphere. In the reference's data model (surface.py:52-119) a
geometry image is a ``SurfaceSamples`` set plus an *identity* quadtree atlas:
one part (``part_count = 1``), ``cell_of = arange(N)`` (row * side + col), no
PAD cells, so ``atlas_flat_cells`` (transfer.py:122-125) is the identity and the
w0 / w1 domains are the S x S grid itself.

This is host-side input generation (like the reference's meshgen.py), not part
of the measured path. Frozen rules:
  * texel (row i, col j) -> (u, v) = ((j + .5)/S, (i + .5)/S) -> octahedral
    decode to a unit direction d;
  * r(d) = R (1 + amp * sum_m sin(k_m . d + phi_m)), m = 1..8, |k_m| ~ U[1, 4]
    along a uniformly random axis, phi_m ~ U[0, 2 pi), seeded;
  * normals analytic: n = normalize(d - grad_s r / r);
  * area = lumped texel area: the texel split into 4 x 4 sub-quads whose
    corners are mapped exactly, each sub-quad two triangles;
  * positions / normals / areas are rounded to float32 (BASELINE: "fp32
    positions, normals and per-point areas"); every consumer reads those.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class GeometryImage:
    side: int
    positions: np.ndarray  # (N, 3) float32, mm
    normals: np.ndarray  # (N, 3) float32, unit
    area: np.ndarray  # (N,) float32, mm^2

    @property
    def count(self) -> int:
        return self.side * self.side

    @property
    def cell_of(self) -> np.ndarray:
        """Identity atlas (surface.py:64-119 with part_count = 1)."""
        return np.arange(self.count, dtype=np.uint32)


def octahedral_decode(u, v):
    """(u, v) in [0,1]^2 -> unit directions (..., 3)."""
    px = 2.0 * np.asarray(u, np.float64) - 1.0
    py = 2.0 * np.asarray(v, np.float64) - 1.0
    nz = 1.0 - np.abs(px) - np.abs(py)
    sx = np.where(px >= 0.0, 1.0, -1.0)
    sy = np.where(py >= 0.0, 1.0, -1.0)
    nx = np.where(nz < 0.0, (1.0 - np.abs(py)) * sx, px)
    ny = np.where(nz < 0.0, (1.0 - np.abs(px)) * sy, py)
    d = np.stack([nx, ny, nz], axis=-1)
    return d / np.linalg.norm(d, axis=-1, keepdims=True)


def _bumps(seed, terms):
    rng = np.random.default_rng(seed)
    axes = rng.standard_normal((terms, 3))
    axes /= np.linalg.norm(axes, axis=1, keepdims=True)
    k = axes * rng.uniform(1.0, 4.0, terms)[:, None]
    phi = rng.uniform(0.0, 2.0 * np.pi, terms)
    return k, phi


def _radius(d, radius, amp, k, phi):
    return radius * (1.0 + amp * np.sin(d @ k.T + phi).sum(axis=-1))


def make_geometry_image(side: int, radius: float = 10.0, amp: float = 0.05,
                        terms: int = 8, seed: int = 2203) -> GeometryImage:
    if side < 2 or side & (side - 1):
        raise ValueError("geometry-image side must be a power of two >= 2")
    k, phi = _bumps(seed, terms)
    t = (np.arange(side) + 0.5) / side
    v, u = np.meshgrid(t, t, indexing="ij")
    d = octahedral_decode(u, v).reshape(-1, 3)
    r = _radius(d, radius, amp, k, phi)
    pos = d * r[:, None]
    grad = radius * amp * (np.cos(d @ k.T + phi) @ k)
    grad_t = grad - np.sum(grad * d, axis=1, keepdims=True) * d
    nrm = d - grad_t / r[:, None]
    nrm /= np.linalg.norm(nrm, axis=1, keepdims=True)
    # lumped texel areas from exactly-mapped sub-quad corners
    sub = 4
    tc = np.arange(side * sub + 1) / (side * sub)
    vc, uc = np.meshgrid(tc, tc, indexing="ij")
    dc = octahedral_decode(uc, vc)
    pc = dc * _radius(dc.reshape(-1, 3), radius, amp, k, phi).reshape(dc.shape[:2])[..., None]
    p00, p10 = pc[:-1, :-1], pc[:-1, 1:]
    p01, p11 = pc[1:, :-1], pc[1:, 1:]
    tri = (0.5 * np.linalg.norm(np.cross(p10 - p00, p11 - p00), axis=-1)
           + 0.5 * np.linalg.norm(np.cross(p11 - p00, p01 - p00), axis=-1))
    area = tri.reshape(side, sub, side, sub).sum(axis=(1, 3)).reshape(-1)
    return GeometryImage(
        side=side,
        positions=np.ascontiguousarray(pos, np.float32),
        normals=np.ascontiguousarray(nrm, np.float32),
        area=np.ascontiguousarray(area, np.float32),
    )


def from_config(cfg) -> GeometryImage:
    return make_geometry_image(cfg.side, cfg.radius, cfg.bump_amp,
                               cfg.bump_terms, cfg.seed)
