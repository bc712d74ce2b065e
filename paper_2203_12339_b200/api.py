"""The reference's public API seam, on the B200: ``Scene`` and
``precompute_compressed`` with the reference's constructor / function
signatures and semantics (runtime.py:65-227, transfer.py:350-361), for ANY
QuadtreeAtlas (several parts, PAD cells) and the reference's default
wavelets (full-pyramid Haar on w0, CDF 9/7 on w1).

A user of ``sssrelight`` switches by import:

    from paper_2203_12339_b200.api import Scene, precompute_compressed

and passes the objects the reference already built (TriangleMesh,
SurfaceSamples, QuadtreeAtlas, DiffusionBasis, a Container from
``load_container`` or this module's ``load_container``, the RayAccelerator,
OpticalMaterial, LightRig, Camera). Everything per frame runs on the GPU:

  stage 1  sss_direct_irradiance64 (shadow rays through the reference's own
           BVH arrays) -> sss_atlas_scatter -> sss_wavelet2d (Haar, full) ->
           sss_select_topn (exact top-n, flat-index ties); ambient:
           sss_env_project
  stage 2  sss_pack_x_bits + sss_transfer_kfr (deterministic fp64 sums;
           sss_transfer_flat16 beyond 65536 rows), folded operators likewise
  stage 3  sss_material_weights
  stage 4  sss_atlas_recombine
  stage 5  sss_wavelet2d (9/7 inverse, full) + sss_atlas_shade

The geometry-image fast path (``runtime.Scene``: L-level Haar on both sides,
fused epilogue, CUDA graphs) is the benchmarked frame; this module is the
drop-in for containers the reference itself produced. Parity: radiance within
1e-4 of the reference's Scene.relight (tests/test_gpu_api.py), the reference's
own tests/test_runtime.py run against this class by import swap.
"""

from __future__ import annotations

import hashlib
import math
import time
import warnings
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .layout import kfr_layout, flat16_layout
from .runtime import STAGES, FrameResult
from .transfer import TransferOperator

DEFAULT_E_KEEP = 0.25   # runtime.py:33
ENV_COEFF_KEEP = 128    # runtime.py:34
DEFAULT_STEP1_KEEP = 0.01     # transfer.py:33
DEFAULT_STEP2_FRACTION = 0.95  # transfer.py:34
_INV_PI = 1.0 / math.pi


# ---------------------------------------------------------------------------
# reference data model (duck-typed: the reference's own objects work too)
# ---------------------------------------------------------------------------

@dataclass
class CompressedTransfer:
    """transfer.py:75-93."""

    operators: list
    k_count: int
    step1_keep: float
    step2_fraction: float
    domain_size: int

    @property
    def nnz(self) -> int:
        return sum(op.nnz for op in self.operators)

    @property
    def step1_entries(self) -> int:
        return sum(op.step1_entries for op in self.operators)

    def compression_ratio(self) -> float:
        s1 = self.step1_entries
        return self.nnz / s1 if s1 else 1.0


@dataclass(frozen=True)
class QuadtreeAtlas:
    """The fields of surface.QuadtreeAtlas (surface.py:64-84) a frame uses."""

    part_count: int
    grid_side: int
    part_of: np.ndarray
    cell_of: np.ndarray

    @property
    def cells_per_part(self) -> int:
        return self.grid_side * self.grid_side

    @property
    def sample_count(self) -> int:
        return int(self.part_of.shape[0])


@dataclass
class Container:
    """container.Container (container.py:140-150) as load_container returns it."""

    basis: object
    atlas: QuadtreeAtlas
    compressed: CompressedTransfer
    mesh_hash: bytes
    visibility: object = None
    folded: object = None
    metadata: dict = field(default_factory=dict)


def load_container(path) -> Container:
    """A PRTS1 file (container.py:156-235 layout, prts1.load_prts1) as the
    reference's Container shape."""
    from .prts1 import load_prts1

    c = load_prts1(path)
    atlas = QuadtreeAtlas(c.part_count, c.grid_side, c.part_of, c.cell_of)
    ct = CompressedTransfer(c.operators, len(c.operators), c.step1_keep, c.step2_fraction,
                            c.part_count * c.grid_side ** 2)
    return Container(basis=c.basis, atlas=atlas, compressed=ct, mesh_hash=c.mesh_hash,
                     metadata=c.metadata)


def mesh_content_hash(mesh) -> bytes:
    """TriangleMesh.content_hash (surface.py:42-50)."""
    if hasattr(mesh, "content_hash"):
        return mesh.content_hash()
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(mesh.vertices, np.float64).tobytes())
    h.update(np.ascontiguousarray(mesh.normals, np.float64).tobytes())
    h.update(np.ascontiguousarray(mesh.triangles, np.int32).tobytes())
    return h.digest()


def flat_cells_of(atlas) -> np.ndarray:
    """atlas_flat_cells (transfer.py:122-125)."""
    return (np.asarray(atlas.part_of, np.int64) * atlas.grid_side * atlas.grid_side
            + np.asarray(atlas.cell_of, np.int64))


def _level(side: int) -> int:
    return int(side).bit_length() - 1


# ---------------------------------------------------------------------------
# device forms
# ---------------------------------------------------------------------------

@dataclass
class _Csr:
    """Rows of reference CSC operators (w0 columns -> w1 rows), the fields
    layout.kfr_layout / flat16_layout read. Row / column ids are flat (the
    full-pyramid "tile-major" order of one part is its flat order)."""

    K: int
    n: int
    levels: int
    rowptr: torch.Tensor
    cols: torch.Tensor
    vals: torch.Tensor


def csr_from_operators(operators, n: int, levels: int, device="cuda") -> _Csr:
    """CSC -> row-major with ascending columns in each row (transposed on the
    device), values rounded to f32 as the container stores them."""
    dev = torch.device(device)
    rowptrs, cols_all, vals_all = [], [], []
    base = 0
    for op in operators:
        cp = torch.as_tensor(np.asarray(op.colptr, np.int64), device=dev)
        cid = torch.as_tensor(np.asarray(op.cols, np.int64), device=dev)
        ri = torch.as_tensor(np.asarray(op.rowidx, np.int64), device=dev)
        v = torch.as_tensor(np.asarray(op.vals, np.float64), device=dev).to(torch.float32)
        if ri.numel() and int(ri.max()) >= n:
            raise ValueError("operator row index outside the domain")
        ecol = torch.repeat_interleave(cid, cp[1:] - cp[:-1])
        order = torch.argsort(ri * n + ecol)
        rp = torch.zeros(n + 1, dtype=torch.int64, device=dev)
        rp[1:] = torch.cumsum(torch.bincount(ri, minlength=n), 0)
        rowptrs.append(rp + base)
        cols_all.append(ecol[order].to(torch.int32))
        vals_all.append(v[order])
        base += int(ri.numel())
    return _Csr(K=len(operators), n=n, levels=levels, rowptr=torch.stack(rowptrs),
                cols=torch.cat(cols_all) if cols_all else torch.empty(0, dtype=torch.int32, device=dev),
                vals=torch.cat(vals_all) if vals_all else torch.empty(0, dtype=torch.float32, device=dev))


class _Transfer:
    """One operator set on the device + its frame layout and launcher:
    v (K, 3, n) = T_k x_c for a dense x (3, n) over the column domain."""

    def __init__(self, operators, n: int, levels: int):
        self.n, self.K = n, len(operators)
        csr = csr_from_operators(operators, n, levels)
        self.kind = "kfr" if (self.K <= 16 and n <= 65536) else "flat16"
        nsm = torch.cuda.get_device_properties(0).multi_processor_count
        # the geometry-image runtime's kfr configuration (8-step batches, 2
        # CTAs/SM, chunk length from the operator)
        self.lay = (kfr_layout(csr, chunk=0, steps_per_batch=8, n_warps=nsm * 2 * 8)
                    if self.kind == "kfr" else flat16_layout(csr))
        dev = torch.device("cuda")
        self.xp = torch.empty((n, 4), dtype=torch.float64, device=dev)
        self.xbits = torch.zeros((n >> 5) + 1, dtype=torch.int32, device=dev)
        self.wctr = torch.zeros(1, dtype=torch.int32, device=dev)
        self.nsm = torch.cuda.get_device_properties(0).multi_processor_count

    def _flat16_partials(self, ne: int, E: int) -> torch.Tensor:
        """Per-word partial sums of the deterministic flat16 form."""
        if getattr(self, "_f16_part", None) is None:
            self._f16_part = torch.zeros(((ne // E + 31) // 32, 6), dtype=torch.float64,
                                         device="cuda")
        return self._f16_part

    def apply(self, x: torch.Tensor, vk: torch.Tensor, sp):
        _lib.call("sss_pack_x_bits", _lib.ptr(x), self.n, _lib.ptr(self.xp), _lib.ptr(self.xbits), sp)
        if self.kind == "kfr":
            lay = self.lay
            _lib.call("sss_transfer_kfr", self.K, self.n, lay.n_items, lay.n_partials,
                      _lib.ptr(lay.items), _lib.ptr(lay.lane_len), _lib.ptr(lay.lane_dst),
                      _lib.ptr(lay.batch_off), _lib.ptr(lay.stream), _lib.ptr(self.xp),
                      _lib.ptr(self.xbits), _lib.ptr(vk), _lib.ptr(lay.partials),
                      _lib.ptr(lay.partial_row), _lib.ptr(lay.multi_info), _lib.ptr(lay.multi_count),
                      _lib.ptr(lay.work), lay.stats["steps_per_batch"], self.nsm * 2 * 8, 2, sp)
        else:
            pcols, pvals, ne, heads, hpre, rowk, wbeg, W, st = self.lay
            _lib.call("sss_zero", _lib.ptr(self.wctr), 4, sp)
            _lib.call("sss_transfer_flat16", self.K, self.n, _lib.ptr(pcols), _lib.ptr(pvals), ne,
                      _lib.ptr(heads), _lib.ptr(hpre), _lib.ptr(rowk), _lib.ptr(wbeg), W, 8, st["E"],
                      st["col_bits"], 1, _lib.ptr(self.xp), _lib.ptr(self.xbits), _lib.ptr(vk),
                      _lib.ptr(self.wctr), 4, _lib.ptr(self._flat16_partials(ne, st["E"])),
                      _lib.ptr(st["span_first"]), sp)


def pack_accelerator(accel):
    """The reference RayAccelerator's arrays (lighting.py:101-170) as the
    GPU BVH records of sss_direct_irradiance (shadows.BVH.packed layout):
    the same tree, so the same any-hit answers."""
    from .shadows import BVH

    b = BVH(np.asarray(accel.node_min, np.float64), np.asarray(accel.node_max, np.float64),
            np.asarray(accel.node_left, np.int32), np.asarray(accel.node_right, np.int32),
            np.asarray(accel.node_start, np.int32), np.asarray(accel.node_count, np.int32),
            np.asarray(accel.v0, np.float64), np.asarray(accel.e1, np.float64),
            np.asarray(accel.e2, np.float64), float(accel.bbox_diagonal), float(accel.ray_offset))
    if b.node_min.shape[0] == 0:
        return None, b
    return b.packed(), b


def pack_lights(rig):
    """(n, 12) light records + kinds for sss_direct_irradiance from a LightRig
    (the reference's classes or shadows.py's: matched by type name)."""
    direct = list(rig.direct_lights)
    out = np.zeros((max(len(direct), 1), 12))
    for i, l in enumerate(direct):
        name = type(l).__name__
        if name == "PointLight":
            out[i, 0], out[i, 1:4], out[i, 4:7] = 0, l.position, l.intensity
        elif name == "DirectionalLight":
            out[i, 0], out[i, 1:4], out[i, 4:7] = 1, l.direction, l.irradiance
        elif name == "SphereLight":
            out[i, 0], out[i, 1:4], out[i, 4:7], out[i, 7] = 2, l.center, l.radiance, l.radius
        else:
            raise TypeError(f"unsupported light {name}")
    return out, out[: len(direct), 0].astype(np.int32)


def _ambient_faces(amb):
    env = getattr(amb, "environment", amb)
    return np.asarray(env.faces, np.float64)


# ---------------------------------------------------------------------------
# Scene (runtime.py:65-227)
# ---------------------------------------------------------------------------

class Scene:
    """Owns the full relight state and the stage-2 cache for fast edits, in
    HBM. Reference signature and semantics (runtime.py:65-227)."""

    def __init__(self, mesh, samples, container, accel, material, rig, camera,
                 e_keep: float = DEFAULT_E_KEEP):
        if container.mesh_hash != mesh_content_hash(mesh):
            raise ValueError("container was precomputed for a different mesh")
        if container.atlas.sample_count != samples.count:
            raise ValueError("sample count mismatch between container and mesh")
        _lib.load()
        self.mesh = mesh
        self.samples = samples
        self.container = container
        self.accel = accel
        self.rig = rig
        self.camera = camera
        self.e_keep = e_keep
        self.material = self._clamp_material(material)
        atlas = container.atlas
        self._side = int(atlas.grid_side)
        self._m = int(atlas.part_count)
        self._D = int(container.compressed.domain_size)
        if self._D != self._m * self._side ** 2:
            raise ValueError("container domain does not match its atlas")
        self._n = int(samples.count)
        dev = torch.device("cuda")
        f64 = dict(dtype=torch.float64, device=dev)
        self._flat = torch.as_tensor(flat_cells_of(atlas).astype(np.int32), device=dev)
        self._pos = torch.as_tensor(np.ascontiguousarray(samples.positions, np.float64), device=dev)
        self._nrm = torch.as_tensor(np.ascontiguousarray(samples.normals, np.float64), device=dev)
        packed, self._bvh = pack_accelerator(accel)
        self._nodes = None if packed is None else torch.as_tensor(packed[0], device=dev)
        self._tris = None if packed is None else torch.as_tensor(packed[1], device=dev)
        self._transfer = _Transfer(container.compressed.operators, self._D, _level(self._side))
        self._folded = None
        self._K = int(container.compressed.k_count)
        b = container.basis
        w = np.empty_like(np.asarray(b.r_nodes, np.float64))  # trapezoid_weights, basisgen.py:90-95
        r = np.asarray(b.r_nodes, np.float64)
        w[0], w[-1] = (r[1] - r[0]) / 2.0, (r[-1] - r[-2]) / 2.0
        w[1:-1] = (r[2:] - r[:-2]) / 2.0
        self._bw = torch.as_tensor(np.ascontiguousarray(np.asarray(b.bases) * w), device=dev)
        self._rn = torch.as_tensor(r, device=dev)
        self._E = torch.empty((3, self._n), **f64)
        self._grid = torch.empty((3, self._D), **f64)
        self._x = torch.empty((3, self._D), **f64)
        self._mask = torch.empty((3, (self._D + 31) // 32), dtype=torch.int32, device=dev)
        self._energy = torch.zeros((3, 2), **f64)
        self._vk = torch.empty((self._K, 3, self._D), **f64)
        self._vk_amb = None
        self._g = torch.empty((3, self._K), **f64)
        self._mat = torch.empty(7, **f64)
        self._cam = torch.empty(3, **f64)
        self._rad = torch.empty((2, self._n, 3), **f64)
        self._vk_cache = None
        self._cache_energy = 0.0

    @property
    def basis(self):
        return self.container.basis

    def _clamp_material(self, material):
        """runtime.py:92-103."""
        from .basis import OpticalMaterial

        lo_p, hi_p, lo_a, hi_a = self.container.basis.sigma_box
        sp = np.clip(material.sigma_s_prime, lo_p, hi_p)
        sa = np.clip(material.sigma_a, lo_a, hi_a)
        if not (np.array_equal(sp, material.sigma_s_prime)
                and np.array_equal(sa, material.sigma_a)):
            warnings.warn("material clamped to the basis sigma box", stacklevel=3)
            cls = type(material)
            try:
                return cls(sigma_s_prime=sp, sigma_a=sa, g=material.g, eta=material.eta)
            except TypeError:
                return OpticalMaterial(sigma_s_prime=sp, sigma_a=sa, g=material.g, eta=material.eta)
        return material

    def _upload(self, dst: torch.Tensor, host):
        dst.copy_(torch.as_tensor(np.asarray(host, np.float64).reshape(dst.shape)))

    # ------------------------------------------------------------------
    # stages
    # ------------------------------------------------------------------

    def _stage1(self, sp, E=None):
        m = self.material
        self._upload(self._mat, np.concatenate([m.sigma_s_prime, m.sigma_a, [m.eta]]))
        lights, kinds = pack_lights(self.rig)
        n_direct = len(kinds)
        if E is not None:  # parity hook: a given (N, 3) irradiance
            self._E.copy_(torch.as_tensor(np.ascontiguousarray(np.asarray(E, np.float64).T)))
        elif n_direct and self._nodes is not None:
            L = torch.as_tensor(lights, device="cuda")
            _lib.call("sss_direct_irradiance64", self._n, _lib.ptr(self._pos), _lib.ptr(self._nrm),
                      n_direct, _lib.ptr(torch.as_tensor(kinds)), _lib.ptr(L), _lib.ptr(self._mat),
                      float(self._bvh.ray_offset), float(self._bvh.bbox_diagonal),
                      _lib.ptr(self._nodes), _lib.ptr(self._tris), _lib.ptr(self._E), sp)
        elif n_direct:  # empty mesh BVH: nothing shadows (_kernels_nb.py:269-270)
            raise ValueError("direct lights need a non-empty RayAccelerator")
        else:
            self._E.zero_()
        _lib.call("sss_atlas_scatter", _lib.ptr(self._E), 3, self._n, _lib.ptr(self._flat), self._D,
                  _lib.ptr(self._grid), sp)
        _lib.call("sss_wavelet2d", _lib.ptr(self._grid), _lib.ptr(self._grid), 3 * self._m,
                  self._side, 0, 0, 0, sp)
        keep = max(1, int(round(self.e_keep * self._D)))  # runtime.py:112
        _lib.call("sss_select_topn", _lib.ptr(self._grid), 3, self._D, keep, None, _lib.ptr(self._x),
                  _lib.ptr(self._mask), _lib.ptr(self._energy), sp)
        amb = self.rig.ambient
        env = None
        if amb is not None:  # runtime.py:120-135
            folded = self.container.folded
            if folded is None:
                raise ValueError("container lacks folded visibility; "
                                 "precompute with --ambient to light environments")
            if abs(folded.eta - self.material.eta) > 1e-9:
                warnings.warn("folded ambient operator was baked for eta="
                              f"{folded.eta:g}; ambient response uses that Fresnel weighting",
                              stacklevel=3)
            faces = _ambient_faces(amb)
            if faces.shape[1] != folded.face_side:
                raise ValueError(f"environment face side {faces.shape[1]} "
                                 f"!= folded operator side {folded.face_side}")
            env = self._project_environment(faces, sp)
        return env

    def _project_environment(self, faces, sp):
        """project_environment (lighting.py:293-305) on the device: the kept
        w2 spectrum of each channel, dense over the folded operators' columns."""
        s = faces.shape[1]
        W = 6 * s * s
        dev = torch.device("cuda")
        fd = torch.as_tensor(np.ascontiguousarray(faces), device=dev)
        kk = min(ENV_COEFF_KEEP, W)
        idx = torch.empty((3, kk), dtype=torch.int32, device=dev)
        val = torch.empty((3, kk), dtype=torch.float64, device=dev)
        _lib.call("sss_env_project", _lib.ptr(fd), s, kk, _lib.ptr(idx), _lib.ptr(val), None, None,
                  None, sp)
        return idx, val, W

    def _ensure_folded(self, W):
        if self._folded is None or self._folded.n != max(self._D, W):
            n = max(self._D, W)  # kfr: square index space (columns < n)
            self._folded = _Transfer(self.container.folded.operators, n, _level(self._side))
            self._xenv = torch.empty((3, n), dtype=torch.float64, device="cuda")
            self._vk_amb_full = torch.empty((self._K, 3, n), dtype=torch.float64, device="cuda")
        return self._folded

    def _stage2(self, env, sp):
        self._transfer.apply(self._x, self._vk, sp)
        self._vk_amb = None
        if env is not None:
            idx, val, W = env
            ft = self._ensure_folded(W)
            self._xenv.zero_()
            ok = idx >= 0
            for c in range(3):
                self._xenv[c].index_copy_(0, idx[c][ok[c]].long(), val[c][ok[c]])
            ft.apply(self._xenv, self._vk_amb_full, sp)
            self._vk_amb = self._vk_amb_full[:, :, : self._D].contiguous()

    def _finish_device(self, ev=None):
        sp = _lib.stream_ptr()
        _lib.call("sss_material_weights", _lib.ptr(self._bw), _lib.ptr(self._rn), self._K,
                  self._rn.numel(), _lib.ptr(self._mat), _lib.ptr(self._g), sp)
        _lib.call("sss_atlas_recombine", self._K, self._D, _lib.ptr(self._vk),
                  _lib.ptr(self._vk_amb), _lib.ptr(self._g), _lib.ptr(self._grid), sp)
        if ev:
            ev[0].record()
        _lib.call("sss_wavelet2d", _lib.ptr(self._grid), _lib.ptr(self._grid), 3 * self._m,
                  self._side, 0, 1, 1, sp)
        self._upload(self._cam, self.camera.position)
        _lib.call("sss_atlas_shade", self._n, self._D, _lib.ptr(self._grid), _lib.ptr(self._flat),
                  _lib.ptr(self._pos), _lib.ptr(self._nrm), _lib.ptr(self._cam), _lib.ptr(self._mat),
                  _lib.ptr(self._rad[0]), _lib.ptr(self._rad[1]), sp)

    # ------------------------------------------------------------------
    # public operations (runtime.py:174-227)
    # ------------------------------------------------------------------

    def relight(self) -> FrameResult:
        """Full pipeline; repopulates the stage-2 cache."""
        return self._relight()

    def relight_from_irradiance(self, E) -> FrameResult:
        """Parity hook: the frame for a given direct irradiance E (N, 3)
        instead of the rig's (stages 1b-5 unchanged)."""
        return self._relight(E)

    def _relight(self, E=None) -> FrameResult:
        timings = dict.fromkeys(STAGES, 0.0)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        sp = _lib.stream_ptr()
        ev[0].record()
        env = self._stage1(sp, E)
        ev[1].record()
        self._stage2(env, sp)
        ev[2].record()
        ev[2].synchronize()
        timings["irradiance"] = ev[0].elapsed_time(ev[1])
        timings["transfer"] = ev[1].elapsed_time(ev[2])
        e = self._energy.cpu().numpy()
        total, kept = float(e[:, 0].sum()), float(e[:, 1].sum())
        self._cache_energy = kept / total if total else 1.0
        self._vk_cache = self._vk
        return self._finish(timings)

    def set_material(self, material) -> FrameResult:
        """Fast edit path: stages 3-5 only, against the cached transfer."""
        if self._vk_cache is None:
            self.material = self._clamp_material(material)
            return self.relight()
        eta_changed = material.eta != self.material.eta
        self.material = self._clamp_material(material)
        if eta_changed and self.rig.direct_lights:
            return self.relight()  # incident Fresnel weighting lives inside E
        m = self.material
        self._upload(self._mat, np.concatenate([m.sigma_s_prime, m.sigma_a, [m.eta]]))
        return self._finish(dict.fromkeys(STAGES, 0.0))

    def _finish(self, timings) -> FrameResult:
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        ev[0].record()
        self._finish_device(ev[1:])
        ev[2].record()
        out = self._rad.cpu().numpy()  # synchronizes
        timings["weighting"] = ev[0].elapsed_time(ev[1])
        timings["inverse_wavelet"] = ev[1].elapsed_time(ev[2])
        return FrameResult(radiance=out[0], radiance_unclamped=out[1], timings_ms=timings,
                           kept_energy_ratio=self._cache_energy)

    def set_light(self, rig) -> FrameResult:
        self.rig = rig
        return self.relight()

    def set_camera(self, camera) -> FrameResult:
        """Camera only affects shading and raster; reuse the cache."""
        self.camera = camera
        if self._vk_cache is None:
            return self.relight()
        return self._finish(dict.fromkeys(STAGES, 0.0))

    def selected_indices(self, c: int) -> np.ndarray:
        """Kept w0 ids of channel c's irradiance spectrum (parity hook)."""
        words = self._mask[c].cpu().numpy().view(np.uint32)
        bits = np.unpackbits(words.view(np.uint8), bitorder="little")[: self._D]
        return np.flatnonzero(bits).astype(np.uint32)


# ---------------------------------------------------------------------------
# precompute_compressed (transfer.py:185-361)
# ---------------------------------------------------------------------------

def _rows_block(ids, pos_d, pos_f64, area_d, rn, bs, sl, K, n, out):
    blk = pos_d[ids]
    _lib.call("sss_transfer_rows", ids.numel(), n, K, rn.numel(), int(pos_f64), _lib.ptr(blk),
              _lib.ptr(pos_d), _lib.ptr(area_d), _lib.ptr(rn), _lib.ptr(bs), _lib.ptr(sl),
              _lib.ptr(out), _lib.stream_ptr())


def precompute_compressed(samples, atlas, basis, step1_keep: float = DEFAULT_STEP1_KEEP,
                          step2_fraction: float = DEFAULT_STEP2_FRACTION, spill_dir=None,
                          progress=None, block_rows: int = None) -> CompressedTransfer:
    """The two-step compression (transfer.py:185-361) on the GPU for any
    atlas, full-pyramid Haar on w0 and CDF 9/7 on w1, bitwise the reference's
    arithmetic: transfer rows (sss_transfer_rows), scatter to the part grids,
    Haar, per-row top-n (stable |v| order, lower flat index first) -> per-k
    unions; a second pass re-derives the union columns (f32), 9/7 along the
    receivers, per-column energy cut with the reference's sequential cumsum
    (sss_energy_cut). The operators (and their kept index sets) are those
    the reference builds. spill_dir is accepted for signature compatibility
    (the unions live in HBM)."""
    if not 0.0 <= step2_fraction <= 1.0:
        raise ValueError("fraction must be in [0, 1]")
    _lib.load()
    dev = torch.device("cuda")
    n = int(samples.count)
    side, m = int(atlas.grid_side), int(atlas.part_count)
    D = m * side * side
    K = int(basis.K)
    n_keep = max(int(round(step1_keep * D)), 1)  # transfer.py:220
    if n_keep < 1:
        raise ValueError("step-1 n must be >= 1")
    keep = min(n_keep, D)
    flat = torch.as_tensor(flat_cells_of(atlas).astype(np.int32), device=dev)
    pos = np.asarray(samples.positions)
    pos_f64 = pos.dtype != np.float32
    pos_d = torch.as_tensor(np.ascontiguousarray(pos, np.float64 if pos_f64 else np.float32),
                            device=dev)
    area_d = torch.as_tensor(np.asarray(samples.area, np.float64), device=dev)
    r_nodes = np.asarray(basis.r_nodes, np.float64)
    bases = np.asarray(basis.bases, np.float64)
    slopes = (bases[:, 1:] - bases[:, :-1]) / np.diff(r_nodes)  # transfer.py:158-159
    rn = torch.as_tensor(r_nodes, device=dev)
    bs = torch.as_tensor(np.ascontiguousarray(bases), device=dev)
    sl = torch.as_tensor(np.ascontiguousarray(slopes), device=dev)
    if block_rows is None:  # (B K, D) f64 spectra + the sort's keys / indices
        block_rows = max(1, min(n, (1 << 25) // max(K * D, 1)))
    sp = _lib.stream_ptr()

    def spectra(ids):
        rows = torch.empty((ids.numel(), K, n), dtype=torch.float64, device=dev)
        _rows_block(ids, pos_d, pos_f64, area_d, rn, bs, sl, K, n, rows)
        buf = torch.empty((ids.numel() * K, D), dtype=torch.float64, device=dev)
        _lib.call("sss_atlas_scatter", _lib.ptr(rows), ids.numel() * K, n, _lib.ptr(flat), D,
                  _lib.ptr(buf), sp)
        _lib.call("sss_wavelet2d", _lib.ptr(buf), _lib.ptr(buf), ids.numel() * K * m, side, 0, 0, 0,
                  sp)
        return buf.view(ids.numel(), K, D)

    # pass 1: step-1 top-n per (row, k) -> unions (run_step1 + step1_unions)
    union = torch.zeros((K, D), dtype=torch.bool, device=dev)
    for lo in range(0, n, block_rows):
        ids = torch.arange(lo, min(lo + block_rows, n), device=dev)
        co = spectra(ids)
        order = torch.sort(-co.abs(), dim=2, stable=True).indices[:, :, :keep]
        for k in range(K):
            union[k].index_fill_(0, order[:, k].reshape(-1), True)
        del co, order
        if progress:
            progress(int(ids[-1]) + 1, n)
    col_ids = [torch.nonzero(union[k]).flatten() for k in range(K)]
    step1_entries = [n * keep] * K
    # pass 2: the union columns' true coefficients, f32 (compress_step2)
    columns = [torch.empty((c.numel(), n), dtype=torch.float32, device=dev) for c in col_ids]
    for lo in range(0, n, block_rows):
        ids = torch.arange(lo, min(lo + block_rows, n), device=dev)
        co = spectra(ids)
        for k in range(K):
            columns[k][:, lo:lo + ids.numel()] = co[:, k, col_ids[k]].T.to(torch.float32)
        del co
    ops = [_threshold_columns(columns[k], col_ids[k], flat, m, side, D, step2_fraction,
                              step1_entries[k]) for k in range(K)]
    del columns
    return CompressedTransfer(operators=ops, k_count=K, step1_keep=step1_keep,
                              step2_fraction=step2_fraction, domain_size=D)


def _threshold_columns(column_values, cols, flat, m, side, D, fraction, step1_entries):
    """transfer.py:303-333 + compress_energy (wavelets.py:139-153) per
    column, on the device: 9/7 of the column over the part grids, stable
    descending-|v| order, the sequential-cumsum cut (sss_energy_cut), kept
    ids ascending. Energies: sum of squares per column (bookkeeping)."""
    dev = column_values.device
    n = column_values.shape[1]
    U = column_values.shape[0]
    chunk = max(1, min(max(U, 1), (1 << 24) // max(D, 1)))
    counts, rows_all, vals_all = [], [], []
    kept_e = total_e = 0.0
    sp = _lib.stream_ptr()
    for c0 in range(0, U, chunk):
        c1 = min(c0 + chunk, U)
        nb = c1 - c0
        batch = torch.empty((nb, D), dtype=torch.float64, device=dev)
        src = column_values[c0:c1].to(torch.float64).contiguous()
        _lib.call("sss_atlas_scatter", _lib.ptr(src), nb, n, _lib.ptr(flat), D, _lib.ptr(batch), sp)
        _lib.call("sss_wavelet2d", _lib.ptr(batch), _lib.ptr(batch), nb * m, side, 0, 1, 0, sp)
        order = torch.sort(-batch.abs(), dim=1, stable=True).indices
        sqT = torch.gather(batch, 1, order).square().T.contiguous()
        nnz = (batch != 0).sum(dim=1).to(torch.int32)
        kept = torch.empty(nb, dtype=torch.int32, device=dev)
        _lib.call("sss_energy_cut", _lib.ptr(sqT), nb, D, float(fraction), _lib.ptr(nnz),
                  _lib.ptr(kept), sp)
        rank_kept = torch.arange(D, device=dev)[None, :] < kept[:, None]
        mask = torch.zeros((nb, D), dtype=torch.bool, device=dev).scatter_(1, order, rank_kept)
        ci, idx = torch.nonzero(mask, as_tuple=True)  # row-major: ids ascending per column
        v = batch[ci, idx]
        tot = batch.square().sum(dim=1)
        kv = torch.zeros(nb, dtype=torch.float64, device=dev).index_add_(0, ci, v * v)
        kept_e += float(torch.minimum(kv, tot).sum())  # wavelets.py:121
        total_e += float(tot.sum())
        counts.append(kept.to(torch.int64))
        rows_all.append(idx.to(torch.int64))
        vals_all.append(v)
        del batch, order, sqT, mask
    colptr = np.zeros(U + 1, np.int64)
    if counts:
        colptr[1:] = torch.cumsum(torch.cat(counts), 0).cpu().numpy()
    return TransferOperator(
        cols=cols.cpu().numpy().astype(np.uint32), colptr=colptr,
        rowidx=(torch.cat(rows_all).cpu().numpy().astype(np.uint32) if rows_all
                else np.empty(0, np.uint32)),
        vals=torch.cat(vals_all).cpu().numpy() if vals_all else np.empty(0, np.float64),
        kept_energy=kept_e, total_energy=total_e, step1_entries=step1_entries)
