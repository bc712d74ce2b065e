"""The per-frame relight / material-edit runtime on one B200.

Mirrors the reference's ``Scene`` (runtime.py:65-227): ``relight``,
``set_material``, ``set_light``, ``set_camera`` -> ``FrameResult`` with the
same fields (radiance, radiance_unclamped, timings_ms over the same STAGES,
kept_energy_ratio, sequence) and the same stage-2 cache semantics: a
material or camera edit re-runs only weights -> recombine -> inverse ->
shade against the cached v_k.

Every stage is a CUDA kernel from ``_sss_b200.so``:
  stage 1  light projection + w0 Haar   sss_sh_irradiance / sss_env_*
           exact top-n                  sss_select_topn
  stage 3  material weights             sss_material_weights (forked stream)
  stage 2  transfer, all K terms and channels at once
                                        sss_pack_x_bits + sss_transfer_kfr
  stage 4+5  recombine + inverse Haar + Fresnel shade
                                        sss_edit_finish
  edit     stages 3-5                   sss_material_weights + sss_edit_finish
The relight sequence can be captured once in a CUDA graph (``capture``)
because every per-frame input (light, material, camera) lives in a device
buffer the kernels read.
"""

from __future__ import annotations

import os
import time
import warnings
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .basis import DiffusionBasis, OpticalMaterial
from .config import CAMERA, E_KEEP, ENV_COEFF_KEEP
from .geometry import GeometryImage
from .lighting import face_directions, face_solid_angles, sh_transfer
from .folding import fold_apply
from .shadows import LightRig, build_bvh, grid_triangles
from .layout import flat16_layout, kfr_layout
from .transfer import DeviceTransfer, flat_to_tile_major

STAGES = ("irradiance", "transfer", "weighting", "inverse_wavelet", "raster")


@dataclass
class Camera:
    """runtime.py:39-53 (position / look_at; only the position shades)."""

    position: np.ndarray
    look_at: np.ndarray = field(default_factory=lambda: np.zeros(3))
    up: np.ndarray = field(default_factory=lambda: np.array([0.0, 1.0, 0.0]))
    fov_y_degrees: float = 40.0

    def __post_init__(self):
        self.position = np.asarray(self.position, np.float64)
        self.look_at = np.asarray(self.look_at, np.float64)
        if np.linalg.norm(self.look_at - self.position) == 0.0:
            raise ValueError("camera position and look-at coincide")
        if not 0.0 < self.fov_y_degrees < 180.0:
            raise ValueError("vertical FOV must lie in (0, 180)")


@dataclass(frozen=True)
class SHLight:
    """Real SH radiance, (bands^2, 3) coefficients per channel."""

    coeffs: np.ndarray

    @property
    def bands(self) -> int:
        return int(round(np.sqrt(self.coeffs.shape[0])))


@dataclass(frozen=True)
class EnvLight:
    """Cubemap radiance (6, s, s, 3), face order +X,-X,+Y,-Y,+Z,-Z."""

    faces: np.ndarray

    @property
    def side(self) -> int:
        return int(self.faces.shape[1])


@dataclass
class FrameResult:
    radiance: np.ndarray  # (N, 3) clamped >= 0
    radiance_unclamped: np.ndarray
    timings_ms: dict
    kept_energy_ratio: float
    sequence: int = 0


class _PinnedBlock:
    """One pinned (2, N, 3) float64 host block lent to a FrameResult: its two
    arrays are numpy views through the buffer protocol, so the block stays
    alive (and out of the pool) until every view of either array is gone."""

    __slots__ = ("pool", "t", "__weakref__")

    def __init__(self, pool, t):
        self.pool, self.t = pool, t

    def __buffer__(self, flags):
        return memoryview(self.t.numpy())

    def __release_buffer__(self, view):
        pass

    def __del__(self):
        self.pool.give_back(self.t)


class _PinnedPool:
    """Recycled pinned read-back blocks for FrameResult arrays. Frames the
    caller keeps hold their blocks; past `cap` blocks outstanding the frame
    falls back to host-converted pageable arrays."""

    def __init__(self, n, cap=64):
        self.n, self.cap, self.free, self.out = n, cap, [], 0

    def take(self):
        if self.free:
            t = self.free.pop()
        elif self.out >= self.cap:
            return None
        else:
            t = torch.empty((2, self.n, 3), dtype=torch.float64, pin_memory=True)
        self.out += 1
        return t

    def give_back(self, t):
        self.out -= 1
        self.free.append(t)


class Scene:
    """Owns the relight state and the stage-2 (v_k) cache, all in HBM."""

    def __init__(self, geometry: GeometryImage, transfer: DeviceTransfer,
                 basis: DiffusionBasis, material: OpticalMaterial, light,
                 camera: Camera = None, e_keep: float = E_KEEP,
                 env_keep: int = ENV_COEFF_KEEP, keep_scatter: bool = False, folded=None):
        _lib.load()
        if transfer.side != geometry.side:
            raise ValueError("transfer operator was precomputed for a different geometry image")
        if transfer.K != basis.K:
            raise ValueError("operator count != basis K")
        self.geometry = geometry
        self.transfer = transfer
        self.folded = folded  # folding.DeviceFolded: the ambient term of a LightRig
        if folded is not None and (folded.side != geometry.side or folded.K != transfer.K or
                                   folded.levels != transfer.levels):
            raise ValueError("folded operators do not match the transfer operators")
        self.basis = basis
        self.e_keep = e_keep
        self.env_keep = env_keep
        self.side, self.levels, self.K = geometry.side, transfer.levels, transfer.K
        n = geometry.count
        self.n = n
        dev = torch.device("cuda")
        f64 = dict(dtype=torch.float64, device=dev)
        self.positions = torch.as_tensor(geometry.positions, device=dev).contiguous()
        self.normals = torch.as_tensor(geometry.normals, device=dev).contiguous()
        self.ehat = torch.empty((3, n), **f64)
        self.x = torch.empty((3, n), **f64)  # masked spectrum, tile-major column order
        self.f2t = torch.as_tensor(
            flat_to_tile_major(np.arange(n), self.side, self.levels).astype(np.int32), device=dev)
        self.mask = torch.empty((3, (n + 31) // 32), dtype=torch.int32, device=dev)
        self.energy = torch.zeros((3, 2), **f64)
        self.g = torch.empty((3, self.K), **f64)
        self.vk = torch.empty((self.K, 3, n), **f64)
        self.radiance = torch.empty((n, 3), dtype=torch.float32, device=dev)
        self.radiance_unclamped = torch.empty((n, 3), dtype=torch.float32, device=dev)
        self.scatter = torch.empty((n, 3), **f64) if keep_scatter else None
        self.E = None
        self.material_buf = torch.empty(7, **f64)
        self.cam_buf = torch.empty(3, **f64)
        self._light_kind = None
        # stage-2 kernel: "kfr" (K-fused row chunks, csrc/transfer.cu; default
        # when K <= 16 and N <= 65536) or "flat16" (flat (row, k)-segment stream,
        # csrc/flat16_25.cu: the A/B alternative and the fallback layout for
        # larger operators). Knobs are read once, here: a captured graph keeps
        # the launch parameters it was recorded with.
        # SSS_TRANSFER=auto (default): both are timed on this operator at the
        # first eager relight and the faster kept (kfr wins on C3-size
        # operators, flat16 on C2's), see _autotune_transfer
        kfr_ok = self.K <= 16 and n <= 65536
        choice = os.environ.get("SSS_TRANSFER", "auto")
        if choice not in ("auto", "kfr", "flat16") or (choice == "kfr" and not kfr_ok):
            raise ValueError(f"unsupported transfer kernel {choice!r}")
        self.transfer_kernel = ("kfr" if kfr_ok else "flat16") if choice == "auto" else choice
        self._autotune = choice == "auto" and kfr_ok
        self.transfer_timings_us = {}
        self._knobs = {
            # kfr: 8-step batches at 2 CTAs/SM, chunk length from the operator
            # (layout.kfr_auto_chunk; 0 = auto). 4 steps / 3 CTAs / 256 was the
            # default until the chunk sweeps (154 vs 142 us on the C3 operator)
            "kfr_chunk": int(os.environ.get("SSS_KFR_CHUNK", "0")),
            "kfr_steps": int(os.environ.get("SSS_KFR_STEPS", "8")),
            "kfr_minb": int(os.environ.get("SSS_KFR_MINB", "2")),
            "flat16_atomics": os.environ.get("SSS_FLAT16_ATOMICS", "0") == "1",
            "env_union_kernel": os.environ.get("SSS_ENV_UNION_KERNEL", "0") == "1",
        }
        self._have_cache = False
        self._sequence = 0
        self._graph = None
        self.camera = camera or Camera(position=np.array(CAMERA[0]))
        self.material = self._clamp_material(material)
        self._write_material()
        self._write_camera()
        self._install_light(light)

    # ------------------------------------------------------------------
    # device-resident inputs
    # ------------------------------------------------------------------

    def _clamp_material(self, material: OpticalMaterial) -> OpticalMaterial:
        """runtime.py:92-103: clip sigma to the basis box with a warning."""
        lo_p, hi_p, lo_a, hi_a = self.basis.sigma_box
        sp = np.clip(material.sigma_s_prime, lo_p, hi_p)
        sa = np.clip(material.sigma_a, lo_a, hi_a)
        if not (np.array_equal(sp, material.sigma_s_prime) and np.array_equal(sa, material.sigma_a)):
            warnings.warn("material clamped to the basis sigma box", stacklevel=3)
            return OpticalMaterial(sigma_s_prime=sp, sigma_a=sa, g=material.g, eta=material.eta)
        return material

    def _write_material(self):
        m = self.material
        self._stage_copy(self.material_buf, np.concatenate([m.sigma_s_prime, m.sigma_a, [m.eta]]))

    def _write_camera(self):
        self._stage_copy(self.cam_buf, self.camera.position)

    def _stage_copy(self, dst: torch.Tensor, host: np.ndarray):
        """Host array -> device buffer through a reused pinned staging tensor.
        The host->device copy is deferred to the next frame submission (one
        call with the frame's graph, sss_frame_replay) or the next eager
        launch (_flush_pending)."""
        key = ("stage", dst.data_ptr())
        pin = getattr(self, "_stage", {}).get(key)
        if pin is None:
            pin = torch.empty(tuple(dst.shape), dtype=dst.dtype, pin_memory=True)
            self._stage = {**getattr(self, "_stage", {}), key: pin}
        # every API frame ends with a synchronize (_frame), so the previous
        # upload from this staging buffer has completed
        pin.numpy()[...] = np.asarray(host, dtype=np.float64).reshape(pin.shape)
        if not hasattr(self, "_pending"):
            self._pending = {}
        self._pending[dst.data_ptr()] = (dst, pin)

    def _flush_pending(self, stream=None):
        """Issue the deferred staging copies on `stream` (eager paths)."""
        pend = getattr(self, "_pending", None)
        if pend:
            with torch.cuda.stream(stream or torch.cuda.current_stream()):
                for dst, pin in pend.values():
                    dst.copy_(pin, non_blocking=True)
            pend.clear()

    def _install_light(self, light):
        dev = torch.device("cuda")
        if isinstance(light, SHLight):
            nl = light.coeffs.shape[0]
            if self._light_kind != ("sh", nl):
                T = sh_transfer(self.geometry.normals, light.bands)  # (N, nl) f32
                self.T_l = torch.as_tensor(np.ascontiguousarray(T.T), device=dev)
                self.light_buf = torch.empty((nl, 3), dtype=torch.float64, device=dev)
                self._light_kind = ("sh", nl)
                self._graph = None
            self._stage_copy(self.light_buf, light.coeffs)
        elif isinstance(light, EnvLight):
            s = light.side
            if self._light_kind != ("env", s):
                D = 6 * s * s
                dirs = torch.as_tensor(face_directions(s).reshape(-1, 3), device=dev)
                dom = torch.as_tensor(face_solid_angles(s).reshape(-1), device=dev)
                self.W2 = torch.empty((D, self.n), dtype=torch.float32, device=dev)
                _lib.call("sss_env_transfer", _lib.ptr(self.normals), self.n, _lib.ptr(dirs),
                          _lib.ptr(dom), s, _lib.ptr(self.W2), _lib.stream_ptr())
                self.light_buf = torch.empty((6, s, s, 3), dtype=torch.float64, device=dev)
                kk = self.env_keep
                self.env_idx = torch.empty((3, kk), dtype=torch.int32, device=dev)
                self.env_val = torch.empty((3, kk), dtype=torch.float64, device=dev)
                self.env_uidx = torch.empty(3 * kk, dtype=torch.int32, device=dev)
                self.env_ulc = torch.empty((3 * kk, 3), dtype=torch.float64, device=dev)
                self.env_nu = torch.empty(1, dtype=torch.int32, device=dev)
                self._light_kind = ("env", s)
                self._graph = None
            self._stage_copy(self.light_buf, light.faces)
        elif isinstance(light, LightRig):
            kinds = tuple(int(k) for k in light.kinds())
            amb = light.ambient
            if amb is not None:  # runtime.py:120-135
                if self.folded is None:
                    raise ValueError("scene lacks folded visibility; build it with "
                                     "folding.fold_visibility to light environments")
                if amb.side != self.folded.face_side:
                    raise ValueError(f"environment face side {amb.side} != folded operator side "
                                     f"{self.folded.face_side}")
                if abs(self.folded.eta - self.material.eta) > 1e-9:
                    warnings.warn(f"folded ambient operator was baked for eta={self.folded.eta:g}; "
                                  "ambient response uses that Fresnel weighting", stacklevel=3)
            amb_side = amb.side if amb is not None else 0
            if self._light_kind != ("direct", kinds, amb_side):
                if getattr(self, "_bvh_dev", None) is None:
                    bvh = build_bvh(self.geometry.positions.astype(np.float64),
                                    grid_triangles(self.side))
                    nodes, tris = bvh.packed()
                    self._bvh_dev = {"nodes": torch.as_tensor(nodes, device=dev),
                                     "tris": torch.as_tensor(tris, device=dev),
                                     "ray_offset": bvh.ray_offset, "diag": bvh.bbox_diagonal}
                self.light_buf = torch.empty((max(len(kinds), 1), 12), dtype=torch.float64,
                                             device=dev)
                self._light_kinds_host = torch.tensor(kinds or (0,), dtype=torch.int32)
                self.E_planar = torch.empty((3, self.n), dtype=torch.float64, device=dev)
                if amb_side:
                    kk = self.env_keep
                    self.amb_buf = torch.empty((6, amb_side, amb_side, 3), dtype=torch.float64,
                                               device=dev)
                    self.env_idx = torch.empty((3, kk), dtype=torch.int32, device=dev)
                    self.env_val = torch.empty((3, kk), dtype=torch.float64, device=dev)
                    self.env_uidx = torch.empty(3 * kk, dtype=torch.int32, device=dev)
                    self.env_ulc = torch.empty((3 * kk, 3), dtype=torch.float64, device=dev)
                    self.env_nu = torch.empty(1, dtype=torch.int32, device=dev)
                self._light_kind = ("direct", kinds, amb_side)
                self._graph = None
            self._n_direct = len(kinds)
            self._stage_copy(self.light_buf, light.packed())
            if amb is not None:
                self._stage_copy(self.amb_buf, amb.faces)
        else:
            raise TypeError(f"unsupported light {type(light).__name__}")
        self.light = light

    # ------------------------------------------------------------------
    # kernel sequences (stream-ordered, capturable)
    # ------------------------------------------------------------------

    def _launch_stage1(self, stream=None, want_E=False, before_select=None, after_project=None):
        sp = _lib.stream_ptr(stream)
        if want_E and self.E is None:
            self.E = torch.empty((self.n, 3), dtype=torch.float64, device="cuda")
        E = self.E if want_E else None
        if self._light_kind[0] == "direct":
            b = self._bvh_dev
            _lib.call("sss_direct_irradiance", self.n, _lib.ptr(self.positions), _lib.ptr(self.normals),
                      self._n_direct, _lib.ptr(self._light_kinds_host), _lib.ptr(self.light_buf),
                      _lib.ptr(self.material_buf), b["ray_offset"], b["diag"], _lib.ptr(b["nodes"]),
                      _lib.ptr(b["tris"]), _lib.ptr(self.E_planar), sp)
            _lib.call("sss_haar2d", _lib.ptr(self.E_planar), _lib.ptr(self.ehat), 3, self.side,
                      self.levels, 0, sp)
            if E is not None:
                E.copy_(self.E_planar.t())
            if self._light_kind[2]:  # the ambient environment's w2 spectrum (runtime.py:135)
                _lib.call("sss_env_project", _lib.ptr(self.amb_buf), self._light_kind[2],
                          self.env_keep, _lib.ptr(self.env_idx), _lib.ptr(self.env_val),
                          _lib.ptr(self.env_uidx), _lib.ptr(self.env_ulc), _lib.ptr(self.env_nu),
                          sp)
        elif self._light_kind[0] == "sh":
            _lib.call("sss_sh_irradiance", _lib.ptr(self.T_l), _lib.ptr(self.light_buf),
                      self._light_kind[1], self.side, self.levels, _lib.ptr(E),
                      _lib.ptr(self.ehat), sp)
        else:
            s, kk = self._light_kind[1], self.env_keep
            if self._knobs["env_union_kernel"]:  # separate union launch
                _lib.call("sss_env_project", _lib.ptr(self.light_buf), s, kk,
                          _lib.ptr(self.env_idx), _lib.ptr(self.env_val), _lib.ptr(self.env_uidx),
                          _lib.ptr(self.env_ulc), _lib.ptr(self.env_nu), sp)
                _lib.call("sss_env_irradiance", _lib.ptr(self.W2), 6 * s * s,
                          _lib.ptr(self.env_uidx), _lib.ptr(self.env_ulc), _lib.ptr(self.env_nu),
                          kk, self.side, self.levels, _lib.ptr(E), _lib.ptr(self.ehat), sp)
            else:  # the union is rebuilt inside every irradiance CTA: one launch less
                _lib.call("sss_env_project", _lib.ptr(self.light_buf), s, kk,
                          _lib.ptr(self.env_idx), _lib.ptr(self.env_val), None, None, None, sp)
                if after_project is not None:
                    after_project()  # forked-stream work joins here, under the projection
                    before_select = lambda: None  # noqa: E731
                _lib.call("sss_env_irradiance_sel", _lib.ptr(self.W2), 6 * s * s,
                          _lib.ptr(self.env_idx), _lib.ptr(self.env_val), kk, self.side,
                          self.levels, _lib.ptr(E), _lib.ptr(self.ehat), sp)
        keep = max(1, int(round(self.e_keep * self.n)))  # runtime.py:112
        # the selection also writes the transfer's inputs (packed x records and
        # the kept-column bitmap): no packing launch. The bitmap is cleared
        # first - on the forked stream when the caller gives the hook
        self._alloc_xp()
        if before_select is not None:
            before_select()
        else:
            _lib.call("sss_zero", _lib.ptr(self.xbits), self.xbits.numel() * 4, sp)
        _lib.call("sss_select_topn_pack", _lib.ptr(self.ehat), self.n, keep, _lib.ptr(self.f2t),
                  _lib.ptr(self.x), _lib.ptr(self.mask), _lib.ptr(self.energy), _lib.ptr(self.xp),
                  _lib.ptr(self.xbits), sp)
        self._x_packed = True

    def _launch_weights(self, stream=None):
        dev = self.basis.device()
        _lib.call("sss_material_weights", _lib.ptr(dev["bw"]), _lib.ptr(dev["r_nodes"]), self.K,
                  len(self.basis.r_nodes), _lib.ptr(self.material_buf), _lib.ptr(self.g),
                  _lib.stream_ptr(stream))

    # ------------------------------------------------------------------
    # stage 2: the scattering transfer (runtime.py:138-150)
    # ------------------------------------------------------------------

    def _transfer_layout(self):
        """The operator copy the frame's transfer kernel reads, built once per
        DeviceTransfer (layout.py)."""
        t = self.transfer
        if self.transfer_kernel == "kfr":
            if getattr(t, "kfr", None) is None:
                nsm = torch.cuda.get_device_properties(0).multi_processor_count
                t.kfr = kfr_layout(t, chunk=self._knobs["kfr_chunk"],
                                   steps_per_batch=self._knobs["kfr_steps"],
                                   n_warps=nsm * self._knobs["kfr_minb"] * 8)
            return t.kfr
        if getattr(t, "flat16", None) is None:
            t.flat16 = flat16_layout(t)
        return t.flat16

    def _alloc_xp(self):
        if getattr(self, "xp", None) is None:
            self.xp = torch.zeros((self.n, 4), dtype=torch.float64, device="cuda")
            self.xbits = torch.zeros((self.n >> 5) + 1, dtype=torch.int32, device="cuda")

    def _pack_x(self, sp):
        """xp (N, 4) f64 + the kept-column bitmap (one clear word past N) from
        self.x - only when x was set some other way than by the frame's
        selection, which writes both itself (sss_select_topn_pack)."""
        self._alloc_xp()
        _lib.call("sss_pack_x_bits", _lib.ptr(self.x), self.n, _lib.ptr(self.xp),
                  _lib.ptr(self.xbits), sp)

    def _transfer_core(self, sp, zero_vk=True):
        lay = self._transfer_layout()
        if self.transfer_kernel == "kfr":
            nsm = torch.cuda.get_device_properties(0).multi_processor_count
            mb = self._knobs["kfr_minb"]
            _lib.call("sss_transfer_kfr", self.K, self.n, lay.n_items, lay.n_partials,
                      _lib.ptr(lay.items), _lib.ptr(lay.lane_len), _lib.ptr(lay.lane_dst),
                      _lib.ptr(lay.batch_off), _lib.ptr(lay.stream),
                      _lib.ptr(self.xp), _lib.ptr(self.xbits), _lib.ptr(self.vk),
                      _lib.ptr(lay.partials), _lib.ptr(lay.partial_row), _lib.ptr(lay.multi_info),
                      _lib.ptr(lay.multi_count), _lib.ptr(lay.work), lay.stats["steps_per_batch"],
                      nsm * mb * 8, mb, sp)
            return
        pcols, pvals, ne, heads, hpre, rowk, wbeg, W, st = lay
        if getattr(self, "_wctr", None) is None:
            self._wctr = torch.zeros(1, dtype=torch.int32, device="cuda")
        # deterministic sums (per-word partials + an ordered merge launch) unless
        # SSS_FLAT16_ATOMICS=1 asks for the fp64-atomics form (A/B)
        part = None
        if not self._knobs["flat16_atomics"]:
            if getattr(self, "_f16_part", None) is None:
                nwords = (ne // st["E"] + 31) // 32
                self._f16_part = torch.zeros((nwords, 6), dtype=torch.float64, device="cuda")
            part = self._f16_part
        _lib.call("sss_transfer_flat16", self.K, self.n, _lib.ptr(pcols), _lib.ptr(pvals), ne,
                  _lib.ptr(heads), _lib.ptr(hpre), _lib.ptr(rowk), _lib.ptr(wbeg), W, 8, st["E"],
                  st["col_bits"], int(zero_vk), _lib.ptr(self.xp), _lib.ptr(self.xbits),
                  _lib.ptr(self.vk), _lib.ptr(self._wctr), 4, _lib.ptr(part),
                  _lib.ptr(st["span_first"]), sp)

    def _autotune_transfer(self, stream=None):
        """Time the core transfer launch of every candidate kernel on this
        operator and this frame's x (CUDA events, 3 launches each after a
        warm-up) and keep the fastest; the other layout is freed. Runs once,
        eagerly (never inside a graph capture)."""
        cands = ["kfr", "flat16"]
        times = {}
        for kern in cands:
            self.transfer_kernel = kern
            self._transfer_layout()
            self.launch_transfer_core(stream)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(3):
                self.launch_transfer_core(stream)
            e1.record(stream)
            e1.synchronize()
            times[kern] = 1e3 * e0.elapsed_time(e1) / 3
        best = min(times, key=times.get)
        self.transfer_kernel = best
        for kern in cands:
            if kern != best:
                setattr(self.transfer, kern, None)
        self.transfer_timings_us = times
        self._autotune = False

    def _launch_transfer(self, stream=None, epilogue=True):
        """Stage 2 (+ stages 3-5 when `epilogue`): v_k = T_k x for every term
        and channel. Returns False: the transfer never fuses the epilogue."""
        sp = _lib.stream_ptr(stream)
        if not getattr(self, "_x_packed", False):
            self._pack_x(sp)
        self._x_packed = False
        if self._autotune and not torch.cuda.is_current_stream_capturing():
            self._autotune_transfer(stream)
        # flat16 accumulates with atomics into a zeroed v_k (zeroed on the side
        # stream by launch_relight when _vk_zeroed); kfr writes every row
        self._transfer_core(sp, zero_vk=not getattr(self, "_vk_zeroed", False))
        if epilogue:
            self._launch_edit(stream)
        return False

    def launch_transfer_core(self, stream=None):
        """The dominant kernel alone, on the inputs the last frame prepared
        (x packed): for roofline timing."""
        sp = _lib.stream_ptr(stream)
        if self.transfer_kernel == "flat16":
            if getattr(self, "_wctr", None) is None:
                self._wctr = torch.zeros(1, dtype=torch.int32, device="cuda")
            _lib.call("sss_zero", _lib.ptr(self._wctr), 4, sp)
            _lib.call("sss_zero", _lib.ptr(self.vk), self.vk.numel() * 8, sp)
        self._transfer_core(sp, zero_vk=False)

    def _launch_edit(self, stream=None):
        # with the API's float64 read-back buffer allocated the epilogue writes
        # the widened pair too (no widening launch per API frame); a graph
        # captured that way says so (_wide)
        r64 = getattr(self, "_rad64", None) if self.levels <= 4 else None
        _lib.call("sss_edit_finish_wide", self.K, self.side, self.levels, _lib.ptr(self.vk),
                  _lib.ptr(self.g), _lib.ptr(self.positions), _lib.ptr(self.normals),
                  _lib.ptr(self.cam_buf), _lib.ptr(self.material_buf), _lib.ptr(self.scatter),
                  _lib.ptr(self.radiance), _lib.ptr(self.radiance_unclamped), _lib.ptr(r64),
                  _lib.stream_ptr(stream))
        return r64 is not None

    def launch_relight(self, stream=None):
        """Enqueue a full relight (no host sync). The material weights do not
        depend on the light: they run on a forked stream, joined before the
        transfer (whose epilogue consumes them), off the stage-1 critical path."""
        cur = stream or torch.cuda.current_stream()
        if not torch.cuda.is_current_stream_capturing():
            self._flush_pending(cur)
        if getattr(self, "_side", None) is None:
            self._side = torch.cuda.Stream()
        fork, join = torch.cuda.Event(), torch.cuda.Event()
        fork.record(cur)
        self._side.wait_event(fork)
        # the kept-column bitmap is cleared on the forked stream too (the
        # selection ORs into it), joined just before the selection
        self._alloc_xp()
        bits_clear = torch.cuda.Event()
        _lib.call("sss_zero", _lib.ptr(self.xbits), self.xbits.numel() * 4,
                  _lib.stream_ptr(self._side))
        bits_clear.record(self._side)
        self._launch_weights(self._side)
        # the default transfer accumulates into a zeroed v_k: zero it here,
        # overlapping stage 1, instead of on the critical path
        self._vk_zeroed = self.transfer_kernel == "flat16"
        if self._vk_zeroed:
            if getattr(self, "_wctr", None) is None:
                self._wctr = torch.zeros(1, dtype=torch.int32, device="cuda")
            _lib.call("sss_zero", _lib.ptr(self.vk), self.vk.numel() * 8, _lib.stream_ptr(self._side))
            _lib.call("sss_zero", _lib.ptr(self._wctr), 4, _lib.stream_ptr(self._side))
        join.record(self._side)
        # environment light + kfr: the forked work (~7 us) ends under the
        # environment projection (~16 us), so it is joined right after that
        # launch and irradiance -> selection -> transfer -> epilogue stay one
        # chain of programmatic dependent launches; otherwise the bitmap clear
        # is joined before the selection and the rest before the transfer
        joined = []

        def join_all():
            cur.wait_event(join)
            joined.append(True)

        self._launch_stage1(cur, before_select=lambda: cur.wait_event(bits_clear),
                            after_project=None if self._vk_zeroed else join_all)
        if not joined:
            cur.wait_event(join)
        if self._ambient_active():
            # v_k = T_k x + F_k L^{w2} (runtime.py:138-150), then stages 3-5
            self._launch_transfer(cur, epilogue=False)
            fold_apply(self.folded, self.env_uidx, self.env_ulc, self.env_nu, self.vk, cur)
            self._launch_edit(cur)
        else:
            self._launch_transfer(cur)
        self._vk_zeroed = False
        self._have_cache = True

    def _ambient_active(self) -> bool:
        return self._light_kind[0] == "direct" and bool(self._light_kind[2])

    def launch_edit(self, stream=None):
        """Enqueue the edit path (no host sync)."""
        if not torch.cuda.is_current_stream_capturing():
            self._flush_pending(stream)
        self._launch_weights(stream)
        self._launch_edit(stream)

    def capture(self):
        """Capture the relight sequence in a CUDA graph (replayed by
        ``replay``); per-frame inputs are the device buffers it reads."""
        if getattr(self, "_pin", None) is None:
            self._enqueue_readback_init()  # the epilogue writes the API's float64 pair
        self.launch_relight()  # warm (sets smem attributes, first-touch)
        torch.cuda.synchronize()
        self._graph_wide = self.levels <= 4
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self.launch_relight()
        self._graph = g
        ge = torch.cuda.CUDAGraph()
        with torch.cuda.graph(ge):
            self.launch_edit()
        self._graph_edit = ge
        return g

    def replay(self, edit=False):
        if self._graph is None:
            self.capture()
        self._flush_pending()
        (self._graph_edit if edit else self._graph).replay()
        self._have_cache = True

    # ------------------------------------------------------------------
    # reference API (runtime.py:174-227)
    # ------------------------------------------------------------------

    def _enqueue_readback_init(self):
        self._pin = {"energy": torch.empty((3, 2), dtype=torch.float64, pin_memory=True),
                     "radu": torch.empty((self.n, 3), dtype=torch.float32, pin_memory=True)}
        self._pool = _PinnedPool(self.n)
        self._rad64 = torch.empty((2, self.n, 3), dtype=torch.float64, device="cuda")

    def _enqueue_readback(self, blk_taken: bool = False):
        """Queue the device->host read-back of the frame's results on the
        current stream, behind the frame's kernels: the radiance and unclamped
        radiance widened to float64 on the device (the reference FrameResult
        dtype) straight into a pooled pinned block that becomes the returned
        arrays, plus the kept-energy sums. No host round trip before the copy,
        no host-side conversion after it."""
        if getattr(self, "_pin", None) is None:
            self._enqueue_readback_init()
        blk = None if blk_taken else self._pool.take()
        if blk is not None:
            _lib.call("sss_widen_frame", _lib.ptr(self.radiance), _lib.ptr(self.radiance_unclamped),
                      self.n * 3, _lib.ptr(self._rad64), _lib.stream_ptr())
            blk.copy_(self._rad64, non_blocking=True)
        else:  # caller holds every pooled block: pageable arrays, host cast
            self._pin["radu"].copy_(self.radiance_unclamped, non_blocking=True)
        self._pin["energy"].copy_(self.energy, non_blocking=True)
        self._blk = blk

    def _frame(self, timings, queued: bool = False) -> FrameResult:
        """One device->host round trip per frame (see _enqueue_readback), one
        synchronize. radiance = max(unclamped, 0) bitwise as on the device."""
        if not queued:
            self._enqueue_readback()
        pin, blk = self._pin, self._blk
        self._blk = None
        torch.cuda.current_stream().synchronize()
        e = pin["energy"].numpy()
        total, kept = float(e[:, 0].sum()), float(e[:, 1].sum())
        self._cache_energy = kept / total if total else 1.0
        self._sequence += 1
        if blk is not None:
            both = np.frombuffer(_PinnedBlock(self._pool, blk), dtype=np.float64).reshape(2, self.n, 3)
            rad, radu = both[0], both[1]
        else:
            u32 = pin["radu"].numpy()
            radu = u32.astype(np.float64)
            rad = np.maximum(u32, 0.0, dtype=np.float64)
        return FrameResult(radiance=rad, radiance_unclamped=radu,
                           timings_ms=timings, kept_energy_ratio=self._cache_energy,
                           sequence=self._sequence)

    def _replay_events(self):
        if getattr(self, "_ev_pair", None) is None:
            self._ev_pair = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
            for e in self._ev_pair:  # create the CUDA events (sss_frame_replay records them)
                e.record()
        return self._ev_pair

    def _submit(self, graph):
        """One API frame's stream work in one library call (sss_frame_replay):
        the deferred staging copies, the start event, the frame's graph, the
        end event, the float64 widening and read-back into a pooled pinned
        block, the kept-energy copy. Returns the start / end events."""
        import ctypes as C

        ev = self._replay_events()
        if getattr(self, "_pin", None) is None:
            self._enqueue_readback_init()
        blk = self._pool.take()
        if blk is None:  # the caller holds every pooled block: the torch path
            self._flush_pending()
            ev[0].record()
            graph.replay()
            ev[1].record()
            self._enqueue_readback(blk_taken=True)
            return ev
        pend = list(self._pending.values()) if getattr(self, "_pending", None) else []
        if pend:
            self._pending.clear()
        n = len(pend)
        wide = getattr(self, "_graph_wide", False)  # the graph's epilogue wrote _rad64
        dsts = (C.c_void_p * max(n, 1))(*[d.data_ptr() for d, _ in pend])
        srcs = (C.c_void_p * max(n, 1))(*[p_.data_ptr() for _, p_ in pend])
        sizes = (C.c_ulonglong * max(n, 1))(*[d.numel() * d.element_size() for d, _ in pend])
        _lib.call("sss_frame_replay", C.c_void_p(graph.raw_cuda_graph_exec()), n, dsts, srcs, sizes,
                  C.c_void_p(ev[0].cuda_event), C.c_void_p(ev[1].cuda_event),
                  None if wide else _lib.ptr(self.radiance),
                  None if wide else _lib.ptr(self.radiance_unclamped), self.n * 3,
                  _lib.ptr(self._rad64), C.c_void_p(blk.data_ptr()), _lib.ptr(self.energy),
                  C.c_void_p(self._pin["energy"].data_ptr()), 48, _lib.stream_ptr())
        self._blk = blk
        return ev

    def relight(self) -> FrameResult:
        """Full pipeline; repopulates the stage-2 cache (runtime.py:174-187).
        The first call runs the kernels eagerly and times every stage
        (irradiance, transfer, weighting, inverse_wavelet = recombine + inverse
        Haar + shade); later calls replay the captured CUDA graph of the same
        sequence and split its measured time by the last eager proportions."""
        timings = dict.fromkeys(STAGES, 0.0)
        # two eager frames first: the first builds the layouts, the second
        # gives steady-state stage proportions for the graph replays
        if self._graph is None and getattr(self, "_eager_relights", 0) >= 2:
            self.capture()
        if self._graph is not None and getattr(self, "_stage_frac", None):
            ev = self._submit(self._graph)
            self._have_cache = True
            fr = self._frame(timings, queued=True)  # synchronizes: ev[1] is complete
            total = ev[0].elapsed_time(ev[1])
            for k, f in self._stage_frac.items():
                timings[k] = total * f
            return fr
        self._eager_relights = getattr(self, "_eager_relights", 0) + 1
        self._flush_pending()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
        ev[0].record()
        self._launch_stage1()
        ev[1].record()
        self._launch_weights()
        ev[2].record()
        self._launch_transfer(epilogue=False)
        if self._ambient_active():
            fold_apply(self.folded, self.env_uidx, self.env_ulc, self.env_nu, self.vk)
        ev[3].record()
        self._launch_edit()
        ev[4].record()
        ev[4].synchronize()
        self._have_cache = True
        timings["irradiance"] = ev[0].elapsed_time(ev[1])
        timings["weighting"] = ev[1].elapsed_time(ev[2])
        timings["transfer"] = ev[2].elapsed_time(ev[3])
        timings["inverse_wavelet"] = ev[3].elapsed_time(ev[4])
        tot = sum(timings.values())
        if tot > 0:
            self._stage_frac = {k: v / tot for k, v in timings.items() if v > 0}
        return self._frame(timings)

    def _edit_frame(self) -> FrameResult:
        timings = dict.fromkeys(STAGES, 0.0)
        if getattr(self, "_graph_edit", None) is not None and self._graph is not None:
            ev = self._submit(self._graph_edit)
            fr = self._frame(timings, queued=True)
            timings["inverse_wavelet"] = ev[0].elapsed_time(ev[1])
            return fr
        self._flush_pending()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        ev[0].record()
        self._launch_weights()
        ev[1].record()
        self._launch_edit()
        ev[2].record()
        ev[2].synchronize()
        timings["weighting"] = ev[0].elapsed_time(ev[1])
        timings["inverse_wavelet"] = ev[1].elapsed_time(ev[2])
        return self._frame(timings)

    def set_material(self, material: OpticalMaterial) -> FrameResult:
        """Fast edit path: stages 3-5 only (runtime.py:189-200). Like the
        reference, an eta change re-runs the full pipeline (the reference's
        irradiance depends on eta; here E is eta-independent by the frozen
        eta_light = 1, so the relight reproduces the same radiance)."""
        if material is self.material and self._have_cache:
            return self._edit_frame()  # unchanged material: nothing to upload
        old_eta = self.material.eta
        self.material = self._clamp_material(material)
        self._write_material()
        if not self._have_cache or self.material.eta != old_eta:
            return self.relight()
        return self._edit_frame()

    def set_light(self, light) -> FrameResult:
        self._install_light(light)
        return self.relight()

    def set_camera(self, camera: Camera) -> FrameResult:
        """Camera only affects shading: reuse the cache (runtime.py:221-226)."""
        self.camera = camera
        self._write_camera()
        if not self._have_cache:
            return self.relight()
        return self._edit_frame()

    # ------------------------------------------------------------------
    # C4: batched material sweep against the cached v_k
    # ------------------------------------------------------------------

    def sweep_prepare(self, materials):
        """Operands of a batched sweep: Bq (3, N, 16) bf16 = w1^-1 v_k of the
        current light, Gq (3, M, 16) bf16 + g64 (M, 3, K) = project_material
        of every material, eta (M) float. Relights first if nothing is cached."""
        if not self._have_cache:
            self.relight()
        if self.K > 16:
            raise ValueError("the sweep supports K <= 16 PCA terms")
        M = len(materials)
        dev = torch.device("cuda")
        mats = np.stack([np.concatenate([self._clamp_material(m).sigma_s_prime,
                                         self._clamp_material(m).sigma_a, [m.eta]])
                         for m in materials]).astype(np.float64)
        eta = mats[:, 6]
        if eta.min() <= 1.0:
            raise ValueError("the sweep needs eta > 1 for every material")
        sp = _lib.stream_ptr()
        ops = {"Bq": torch.empty((3, self.n, 16), dtype=torch.bfloat16, device=dev),
               "Gq": torch.empty((3, M, 16), dtype=torch.bfloat16, device=dev),
               "g64": torch.empty((M, 3, self.K), dtype=torch.float64, device=dev),
               "eta": torch.empty(M, dtype=torch.float32, device=dev),
               "materials": torch.as_tensor(mats, device=dev),
               "eta_range": (float(eta.min()), float(eta.max()))}
        _lib.call("sss_sweep_basis", self.K, self.side, self.levels, _lib.ptr(self.vk),
                  _lib.ptr(ops["Bq"]), sp)
        d = self.basis.device()
        _lib.call("sss_material_weights_batch", _lib.ptr(d["bw"]), _lib.ptr(d["r_nodes"]), self.K,
                  len(self.basis.r_nodes), M, _lib.ptr(ops["materials"]), _lib.ptr(ops["g64"]),
                  _lib.ptr(ops["Gq"]), _lib.ptr(ops["eta"]), sp)
        return ops

    def sweep_launch(self, ops, out, stream=None):
        """out (3, M, N) float32 = clamped exit radiance of every material."""
        self._flush_pending(stream)
        lo, hi = ops["eta_range"]
        _lib.call("sss_sweep_gemm", self.n, ops["Gq"].shape[1], _lib.ptr(ops["Bq"]),
                  _lib.ptr(ops["Gq"]), _lib.ptr(ops["eta"]), lo, hi, _lib.ptr(self.positions),
                  _lib.ptr(self.normals), _lib.ptr(self.cam_buf), _lib.ptr(out),
                  _lib.stream_ptr(stream))

    def sweep(self, materials) -> torch.Tensor:
        """Radiance (3, M, N) of M materials under the current light and camera
        (the C4 batched sweep: one bf16 tcgen05 contraction + Fresnel shade)."""
        ops = self.sweep_prepare(materials)
        out = torch.empty((3, len(materials), self.n), dtype=torch.float32, device="cuda")
        self.sweep_launch(ops, out)
        return out

    def render_image(self, width: int, height: int, exposure: float = 1.0,
                     background=(0.0, 0.0, 0.0)) -> np.ndarray:
        """render_image (runtime.py:230-245) of the current frame's radiance,
        straight from the device buffer (no host round trip of the radiance):
        the geometry image's grid mesh, the scene camera, sRGB u8 out."""
        from .raster import Rasterizer, mesh_of

        key = (int(width), int(height))
        r = getattr(self, "_raster", None)
        if r is None or (r.width, r.height) != key:
            r = self._raster = Rasterizer(mesh_of(self.geometry), width, height)
        return r.render(self.radiance, self.camera, exposure, background)

    # ------------------------------------------------------------------
    # parity hooks
    # ------------------------------------------------------------------

    def selected_indices(self, c: int) -> np.ndarray:
        words = self.mask[c].cpu().numpy().view(np.uint32)
        bits = np.unpackbits(words.view(np.uint8), bitorder="little")[: self.n]
        return np.flatnonzero(bits).astype(np.uint32)


def bench(scene: Scene, iterations: int = 20) -> dict:
    """runtime.py:280-307: median / p10 / p90 of relight and edit (host clock
    around synchronous API calls, like the reference)."""
    if iterations < 1:
        raise ValueError("iterations must be >= 1")
    scene.relight()
    full, edit = [], []
    material = scene.material
    for _ in range(iterations):
        t0 = time.perf_counter()
        scene.relight()
        full.append((time.perf_counter() - t0) * 1e3)
        t0 = time.perf_counter()
        scene.set_material(material)
        edit.append((time.perf_counter() - t0) * 1e3)
    full, edit = np.asarray(full), np.asarray(edit)

    def stats(a):
        return {"median_ms": float(np.median(a)), "p10_ms": float(np.percentile(a, 10)),
                "p90_ms": float(np.percentile(a, 90))}

    return {"iterations": iterations, "relight": stats(full), "material_edit": stats(edit),
            "edit_faster": bool(np.median(edit) < np.median(full))}
