"""Direct lights with shadow rays: the reference's
`irradiance_direct` (lighting.py:208-290) with BVH any-hit visibility
(lighting.py:101-176, _kernels_nb.py:208-298), for geometry images.

Host side: light types mirroring the reference (PointLight, DirectionalLight,
SphereLight, LightRig), the geometry image's grid triangulation, and a
median-split BVH built level by level with numpy (any-hit answers do not
depend on the tree's shape, so it need not match the reference's build
order). The per-sample shadow rays and irradiance run in
`sss_direct_irradiance` on the GPU.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

RAY_OFFSET_SCALE = 1e-4   # lighting.py:23, of the bbox diagonal
SPHERE_LIGHT_SAMPLES = 64  # lighting.py:24
LEAF_SIZE = 4              # lighting.py:22


def _rgb(v) -> np.ndarray:
    return np.broadcast_to(np.asarray(v, np.float64), (3,)).copy()


@dataclass(frozen=True)
class PointLight:
    position: np.ndarray  # mm
    intensity: np.ndarray  # W/sr per channel

    def __post_init__(self):
        object.__setattr__(self, "position", np.asarray(self.position, np.float64))
        object.__setattr__(self, "intensity", _rgb(self.intensity))
        if np.any(self.intensity < 0.0):
            raise ValueError("intensity must be >= 0")


@dataclass(frozen=True)
class DirectionalLight:
    direction: np.ndarray  # light -> scene, normalized on construction
    irradiance: np.ndarray  # W/mm^2 per channel on a facing surface

    def __post_init__(self):
        d = np.asarray(self.direction, np.float64)
        n = np.linalg.norm(d)
        if n == 0.0:
            raise ValueError("direction must be nonzero")
        object.__setattr__(self, "direction", d / n)
        object.__setattr__(self, "irradiance", _rgb(self.irradiance))
        if np.any(self.irradiance < 0.0):
            raise ValueError("irradiance must be >= 0")


@dataclass(frozen=True)
class SphereLight:
    center: np.ndarray  # mm
    radius: float  # mm
    radiance: np.ndarray  # W/(sr mm^2) per channel

    def __post_init__(self):
        object.__setattr__(self, "center", np.asarray(self.center, np.float64))
        object.__setattr__(self, "radiance", _rgb(self.radiance))
        if self.radius < 0.0 or np.any(self.radiance < 0.0):
            raise ValueError("radius and radiance must be >= 0")


@dataclass(frozen=True)
class AmbientLight:
    """An environment cubemap lighting the scene through the folded
    visibility operators (lighting.py:62-64; runtime.py:120-149).
    faces: (6, s, s, 3) radiance."""

    faces: np.ndarray

    def __post_init__(self):
        f = np.asarray(self.faces, np.float64)
        if f.ndim != 4 or f.shape[0] != 6 or f.shape[1] != f.shape[2] or f.shape[3] != 3:
            raise ValueError("faces must be (6, s, s, 3)")
        object.__setattr__(self, "faces", f)

    @property
    def side(self) -> int:
        return int(self.faces.shape[1])


@dataclass(frozen=True)
class LightRig:
    """The lights of a frame (lighting.py:80-98): point / directional /
    sphere lights with shadow rays, plus at most one AmbientLight."""

    lights: tuple

    def __post_init__(self):
        object.__setattr__(self, "lights", tuple(self.lights))
        for l in self.lights:
            if not isinstance(l, (PointLight, DirectionalLight, SphereLight, AmbientLight)):
                raise TypeError(f"unsupported light {type(l).__name__}")
        if sum(isinstance(l, AmbientLight) for l in self.lights) > 1:
            raise ValueError("at most one ambient light")

    @property
    def ambient(self):
        for l in self.lights:
            if isinstance(l, AmbientLight):
                return l
        return None

    @property
    def direct_lights(self) -> list:
        return [l for l in self.lights if not isinstance(l, AmbientLight)]

    def packed(self) -> np.ndarray:
        """(n, 12) doubles per direct light: {kind, a[3], b[3], radius, 0...}; kind 0 =
        point (a = position, b = intensity), 1 = directional (a = unit
        direction, b = irradiance), 2 = sphere (a = center, b = radiance)."""
        direct = self.direct_lights
        out = np.zeros((max(len(direct), 1), 12))
        for i, l in enumerate(direct):
            if isinstance(l, PointLight):
                out[i, 0], out[i, 1:4], out[i, 4:7] = 0, l.position, l.intensity
            elif isinstance(l, DirectionalLight):
                out[i, 0], out[i, 1:4], out[i, 4:7] = 1, l.direction, l.irradiance
            else:
                out[i, 0], out[i, 1:4], out[i, 4:7], out[i, 7] = 2, l.center, l.radiance, l.radius
        return out

    def kinds(self) -> np.ndarray:
        """(n,) int32 kinds in light order (column 0 of packed())."""
        return self.packed()[: len(self.direct_lights), 0].astype(np.int32)


def grid_triangles(side: int) -> np.ndarray:
    """Two triangles per geometry-image cell: (i00, i01, i11), (i00, i11, i10)."""
    r, c = np.meshgrid(np.arange(side - 1), np.arange(side - 1), indexing="ij")
    i00 = (r * side + c).reshape(-1)
    i01, i10 = i00 + 1, i00 + side
    i11 = i10 + 1
    t = np.empty((i00.size * 2, 3), np.int32)
    t[0::2] = np.stack([i00, i01, i11], 1)
    t[1::2] = np.stack([i00, i11, i10], 1)
    return t


@dataclass
class BVH:
    node_min: np.ndarray   # (M, 3) f64
    node_max: np.ndarray   # (M, 3) f64
    node_left: np.ndarray  # (M,) i32, -1 for leaves
    node_right: np.ndarray
    node_start: np.ndarray  # (M,) i32 first triangle (leaves)
    node_count: np.ndarray  # (M,) i32, 0 for inner nodes
    v0: np.ndarray         # (T, 3) f64, triangles in leaf order
    e1: np.ndarray
    e2: np.ndarray
    bbox_diagonal: float
    ray_offset: float

    def packed(self):
        """GPU records (sss_direct_irradiance): nodes (M, 8) f64 = {min[3],
        max[3], i32 (left, right), i32 (start, count)}, tris (T, 10) f64 =
        {v0[3], e1[3], e2[3], 0}."""
        m = self.node_min.shape[0]
        nodes = np.zeros((m, 8), np.float64)
        nodes[:, 0:3], nodes[:, 3:6] = self.node_min, self.node_max
        ints = nodes.view(np.int32)  # (m, 16)
        ints[:, 12], ints[:, 13] = self.node_left, self.node_right
        ints[:, 14], ints[:, 15] = self.node_start, self.node_count
        tris = np.zeros((self.v0.shape[0], 10), np.float64)
        tris[:, 0:3], tris[:, 3:6], tris[:, 6:9] = self.v0, self.e1, self.e2
        return nodes, tris


def _seg_reduce(op, a: np.ndarray, starts: np.ndarray, ends: np.ndarray) -> np.ndarray:
    """op.reduce over a[starts[i]:ends[i]] for disjoint non-empty ranges (any
    order): interleaved [start, end) indices into a padded copy."""
    o = np.argsort(starts, kind="stable")
    idx = np.empty(2 * starts.size, np.int64)
    idx[0::2] = starts[o]
    idx[1::2] = ends[o]
    pad = np.concatenate([a, a[:1]], axis=0)
    red = op.reduceat(pad, idx, axis=0)[0::2]
    out = np.empty_like(red)
    out[o] = red
    return out


def build_bvh(vertices: np.ndarray, tris: np.ndarray, leaf: int = LEAF_SIZE) -> BVH:
    """Median split on the longest centroid axis, built breadth-first with
    segmented sorts (one numpy pass per tree level)."""
    v = np.asarray(vertices, np.float64)
    t = np.asarray(tris, np.int64)
    lo = np.minimum(np.minimum(v[t[:, 0]], v[t[:, 1]]), v[t[:, 2]])
    hi = np.maximum(np.maximum(v[t[:, 0]], v[t[:, 1]]), v[t[:, 2]])
    cen = (lo + hi) / 2.0
    order = np.arange(t.shape[0], dtype=np.int64)
    # frontier: node ids with their [start, end) ranges in `order`
    starts, ends, ids = np.array([0]), np.array([t.shape[0]]), np.array([0])
    total = 1
    rows = {}
    while starts.size:
        # bounds of every frontier node
        bmin = _seg_reduce(np.minimum, lo[order], starts, ends)
        bmax = _seg_reduce(np.maximum, hi[order], starts, ends)
        cnt = ends - starts
        is_leaf = cnt <= leaf
        split = ~is_leaf
        for j in range(ids.size):
            rows[int(ids[j])] = [bmin[j], bmax[j], -1, -1, int(starts[j]) if is_leaf[j] else 0,
                                 int(cnt[j]) if is_leaf[j] else 0]
        if not split.any():
            break
        s_st, s_en, s_id = starts[split], ends[split], ids[split]
        cmin = _seg_reduce(np.minimum, cen[order], s_st, s_en)
        cmax = _seg_reduce(np.maximum, cen[order], s_st, s_en)
        axis = np.argmax(cmax - cmin, axis=1)
        # segmented stable sort of each split node's range by its axis
        seg_len = s_en - s_st
        seg = np.repeat(np.arange(s_st.size), seg_len)
        pos = np.concatenate([np.arange(a, b) for a, b in zip(s_st, s_en)])
        keys = cen[order[pos], axis[seg]]
        o = np.lexsort((keys, seg))
        order[pos] = order[pos][o]
        mid = (s_st + s_en) // 2
        left_ids = total + 2 * np.arange(s_id.size)
        right_ids = left_ids + 1
        total += 2 * s_id.size
        for j in range(s_id.size):
            rows[int(s_id[j])][2] = int(left_ids[j])
            rows[int(s_id[j])][3] = int(right_ids[j])
        starts = np.concatenate([s_st, mid])
        ends = np.concatenate([mid, s_en])
        ids = np.concatenate([left_ids, right_ids])
    M = total
    node_min = np.zeros((M, 3))
    node_max = np.zeros((M, 3))
    node_left = np.full(M, -1, np.int32)
    node_right = np.full(M, -1, np.int32)
    node_start = np.zeros(M, np.int32)
    node_count = np.zeros(M, np.int32)
    for k, (a, b, l, r, s, c) in rows.items():
        node_min[k], node_max[k], node_left[k], node_right[k] = a, b, l, r
        node_start[k], node_count[k] = s, c
    tt = t[order]
    v0 = np.ascontiguousarray(v[tt[:, 0]])
    e1 = np.ascontiguousarray(v[tt[:, 1]] - v[tt[:, 0]])
    e2 = np.ascontiguousarray(v[tt[:, 2]] - v[tt[:, 0]])
    diag = float(np.linalg.norm(v.max(axis=0) - v.min(axis=0)))
    return BVH(node_min, node_max, node_left, node_right, node_start, node_count, v0, e1, e2,
               diag, RAY_OFFSET_SCALE * diag)
