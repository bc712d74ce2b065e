"""Light inputs for path (a): real spherical harmonics and wavelet cubemaps.

Host-side input generation and setup tables only (the per-frame projection
E = T L runs in CUDA, see ``relight.py``).

* SH (configs C1, C2, C4). The reference has no SH light;
  its analogue of path (a) is ``visibility_weights`` + ``ambient_irradiance_
  dense`` (lighting.py:318-336): E = W L with W = V F_t cos+ d_omega. With
  V = 1 and eta_light = 1 (F_t == 1, dipole.py:142-144) the SH transfer is
  T_jl = sum_d W[j, d] Y_l(omega_d) -> the clamped-cosine convolution, which
  Funk-Hecke gives in closed form: T_jl = A_l Y_l(n_j) with A_0 = pi,
  A_1 = 2 pi / 3, A_2 = pi / 4, A_3 = 0, A_4 = -pi / 24. The oracle checks
  the closed form against the reference-anchored cubemap quadrature.
* Cubemap (config C3): face tables follow envmap.py:45-66 (face order
  +X,-X,+Y,-Y,+Z,-Z); the environment is log-normal(0, 1) texels plus three
  Gaussian lobes (peak 50x the log-normal median, 5 deg width); per-frame
  rotation about +y is exact for the lobes and nearest-texel for the
  log-normal layer (frozen).
"""

from __future__ import annotations

import math

import numpy as np

# ---------------------------------------------------------------------------
# real spherical harmonics, bands 0..4 (25 functions), no Condon-Shortley phase
# ---------------------------------------------------------------------------

_PI = math.pi
_SH_CONST = {
    0: [0.5 / math.sqrt(_PI)],
    1: [math.sqrt(3.0 / (4.0 * _PI))] * 3,
    2: [0.5 * math.sqrt(15.0 / _PI), 0.5 * math.sqrt(15.0 / _PI),
        0.25 * math.sqrt(5.0 / _PI), 0.5 * math.sqrt(15.0 / _PI),
        0.25 * math.sqrt(15.0 / _PI)],
    3: [0.25 * math.sqrt(35.0 / (2 * _PI)), 0.5 * math.sqrt(105.0 / _PI),
        0.25 * math.sqrt(21.0 / (2 * _PI)), 0.25 * math.sqrt(7.0 / _PI),
        0.25 * math.sqrt(21.0 / (2 * _PI)), 0.25 * math.sqrt(105.0 / _PI),
        0.25 * math.sqrt(35.0 / (2 * _PI))],
    4: [0.75 * math.sqrt(35.0 / _PI), 0.75 * math.sqrt(35.0 / (2 * _PI)),
        0.75 * math.sqrt(5.0 / _PI), 0.75 * math.sqrt(5.0 / (2 * _PI)),
        (3.0 / 16.0) * math.sqrt(1.0 / _PI), 0.75 * math.sqrt(5.0 / (2 * _PI)),
        (3.0 / 8.0) * math.sqrt(5.0 / _PI), 0.75 * math.sqrt(35.0 / (2 * _PI)),
        (3.0 / 16.0) * math.sqrt(35.0 / _PI)],
}
CLAMPED_COSINE_ZONAL = (_PI, 2.0 * _PI / 3.0, _PI / 4.0, 0.0, -_PI / 24.0)


def sh_band_of(index: int) -> int:
    return int(math.isqrt(index))


def sh_eval(dirs, bands: int) -> np.ndarray:
    """(..., 3) unit directions -> (..., bands^2) real SH values."""
    if not 1 <= bands <= 5:
        raise ValueError("SH bands must lie in [1, 5]")
    d = np.asarray(dirs, np.float64)
    x, y, z = d[..., 0], d[..., 1], d[..., 2]
    x2, y2, z2 = x * x, y * y, z * z
    polys = [
        [np.ones_like(x)],
        [y, z, x],
        [x * y, y * z, 3.0 * z2 - 1.0, x * z, x2 - y2],
        [y * (3.0 * x2 - y2), x * y * z, y * (5.0 * z2 - 1.0),
         z * (5.0 * z2 - 3.0), x * (5.0 * z2 - 1.0), z * (x2 - y2),
         x * (x2 - 3.0 * y2)],
        [x * y * (x2 - y2), y * z * (3.0 * x2 - y2), x * y * (7.0 * z2 - 1.0),
         y * z * (7.0 * z2 - 3.0), 35.0 * z2 * z2 - 30.0 * z2 + 3.0,
         x * z * (7.0 * z2 - 3.0), (x2 - y2) * (7.0 * z2 - 1.0),
         x * z * (x2 - 3.0 * y2), x2 * (x2 - 3.0 * y2) - y2 * (3.0 * x2 - y2)],
    ]
    out = [c * p for l in range(bands) for c, p in zip(_SH_CONST[l], polys[l])]
    return np.stack(out, axis=-1)


def sh_transfer(normals, bands: int) -> np.ndarray:
    """Unshadowed clamped-cosine transfer T (N, bands^2), float32 storage."""
    y = sh_eval(np.asarray(normals, np.float64), bands)
    a = np.array([CLAMPED_COSINE_ZONAL[sh_band_of(i)] for i in range(bands * bands)])
    return np.ascontiguousarray(y * a[None, :], np.float32)


def random_sh_light(bands: int, seed: int) -> np.ndarray:
    """(bands^2, 3): N(0,1)/(1+l)^2 per coefficient and channel, DC > 0."""
    rng = np.random.default_rng(seed)
    L = rng.standard_normal((bands * bands, 3))
    scale = np.array([1.0 / (1.0 + sh_band_of(i)) ** 2 for i in range(bands * bands)])
    L *= scale[:, None]
    L[0] = np.abs(L[0])
    return L


def random_rotation(rng) -> np.ndarray:
    """Uniform on SO(3) (unit quaternion from a normal 4-vector)."""
    q = rng.standard_normal(4)
    q /= np.linalg.norm(q)
    w, x, y, z = q
    return np.array([
        [1 - 2 * (y * y + z * z), 2 * (x * y - z * w), 2 * (x * z + y * w)],
        [2 * (x * y + z * w), 1 - 2 * (x * x + z * z), 2 * (y * z - x * w)],
        [2 * (x * z - y * w), 2 * (y * z + x * w), 1 - 2 * (x * x + y * y)],
    ])


def rotate_sh(L: np.ndarray, R: np.ndarray) -> np.ndarray:
    """Coefficients of f'(w) = f(R^T w), band by band (exact least squares on
    a fixed direction set; each band is rotation-closed)."""
    bands = sh_band_of(L.shape[0] - 1) + 1
    rng = np.random.default_rng(12345)
    w = rng.standard_normal((64, 3))
    w /= np.linalg.norm(w, axis=1, keepdims=True)
    A = sh_eval(w, bands)
    B = sh_eval(w @ R, bands)  # rows: Y(R^T w)
    out = np.zeros_like(L)
    for l in range(bands):
        sl = slice(l * l, (l + 1) * (l + 1))
        M, *_ = np.linalg.lstsq(A[:, sl], B[:, sl], rcond=None)
        out[sl] = M @ L[sl]
    return out


# ---------------------------------------------------------------------------
# cubemaps (envmap.py:45-66 tables; BASELINE C3 environment)
# ---------------------------------------------------------------------------

def face_directions(side: int) -> np.ndarray:
    """(6, s, s, 3) texel directions, envmap.py:45-58."""
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


def face_solid_angles(side: int) -> np.ndarray:
    """(6, s, s), envmap.py:61-66."""
    t = (np.arange(side) + 0.5) / side * 2.0 - 1.0
    v, u = np.meshgrid(t, t, indexing="ij")
    w = 4.0 / (side * side) / np.power(u * u + v * v + 1.0, 1.5)
    return np.tile(w, (6, 1, 1))


def direction_to_texel(dirs, side: int) -> np.ndarray:
    """Nearest texel flat index (face * s * s + row * s + col) for directions,
    inverting face_directions' conventions."""
    d = np.asarray(dirs, np.float64)
    ax = np.abs(d)
    major = np.argmax(ax, axis=-1)
    x, y, z = d[..., 0], d[..., 1], d[..., 2]
    face = np.empty(d.shape[:-1], np.int64)
    u = np.empty(d.shape[:-1])
    v = np.empty(d.shape[:-1])
    m = major == 0
    pos = x > 0
    # +X: (1, -v, -u) ; -X: (-1, -v, u)
    sel = m & pos
    face[sel], u[sel], v[sel] = 0, -z[sel] / ax[sel, 0], -y[sel] / ax[sel, 0]
    sel = m & ~pos
    face[sel], u[sel], v[sel] = 1, z[sel] / ax[sel, 0], -y[sel] / ax[sel, 0]
    m = major == 1
    pos = y > 0
    # +Y: (u, 1, v) ; -Y: (u, -1, -v)
    sel = m & pos
    face[sel], u[sel], v[sel] = 2, x[sel] / ax[sel, 1], z[sel] / ax[sel, 1]
    sel = m & ~pos
    face[sel], u[sel], v[sel] = 3, x[sel] / ax[sel, 1], -z[sel] / ax[sel, 1]
    m = major == 2
    pos = z > 0
    # +Z: (u, -v, 1) ; -Z: (-u, -v, -1)
    sel = m & pos
    face[sel], u[sel], v[sel] = 4, x[sel] / ax[sel, 2], -y[sel] / ax[sel, 2]
    sel = m & ~pos
    face[sel], u[sel], v[sel] = 5, -x[sel] / ax[sel, 2], -y[sel] / ax[sel, 2]
    col = np.clip(np.floor((u + 1.0) * 0.5 * side), 0, side - 1).astype(np.int64)
    row = np.clip(np.floor((v + 1.0) * 0.5 * side), 0, side - 1).astype(np.int64)
    return face * side * side + row * side + col


class Environment:
    """Seeded C3 environment: log-normal layer + 3 Gaussian lobes."""

    def __init__(self, side: int = 32, seed: int = 7, lobes: int = 3,
                 peak: float = 50.0, width_deg: float = 5.0):
        rng = np.random.default_rng(seed)
        self.side = side
        self.base = np.exp(rng.standard_normal((6 * side * side, 3)))  # LN(0,1)
        ld = rng.standard_normal((lobes, 3))
        self.lobe_dirs = ld / np.linalg.norm(ld, axis=1, keepdims=True)
        self.peak = peak  # x the log-normal median (= 1)
        self.sigma = math.radians(width_deg)
        self.dirs = face_directions(side).reshape(-1, 3)

    def faces(self, angle_deg: float = 0.0) -> np.ndarray:
        """(6, s, s, 3) radiance of the environment rotated about +y."""
        a = math.radians(angle_deg)
        c, s = math.cos(a), math.sin(a)
        R = np.array([[c, 0.0, s], [0.0, 1.0, 0.0], [-s, 0.0, c]])
        src = self.dirs @ R  # R^T w: where each texel looks in the base frame
        rad = self.base[direction_to_texel(src, self.side)].copy()
        lobes = self.lobe_dirs @ R.T  # rotated lobe axes (exact)
        cosang = np.clip(self.dirs @ lobes.T, -1.0, 1.0)
        ang = np.arccos(cosang)
        rad += (self.peak * np.exp(-0.5 * (ang / self.sigma) ** 2)).sum(axis=1)[:, None]
        return rad.reshape(6, self.side, self.side, 3)
