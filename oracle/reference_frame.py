"""The reference arm of ``bench.py`` — TEST / BASELINE INFRASTRUCTURE ONLY.

Times the C3 relight / material-edit frame with the REFERENCE's own code
(``sssrelight`` installed under ``baseline/_ref``, numba backend):

* ``container.load_container`` reads the operator (a PRTS1 file the GPU arm
  exported; the reference's own loader, vals f32 -> f64);
* stage 2: ``TransferOperator.apply`` -> ``_kernels_nb.csc_apply`` (numba), the
  K x 3 calls of ``Scene._stage2_transfer`` (runtime.py:138-150);
* ``wavelets.compress_top_n`` (stage 1 selection, runtime.py:112-118),
  ``basisgen.project_material`` (stage 3), the einsum of ``_finish``
  (runtime.py:202-216) and ``dipole.fresnel_transmittance`` in ``_shade``
  (runtime.py:162-168).

Where BASELINE's C3 changes the operation the reference has no code for, the
oracle's restatements fill in (oracle/sss_oracle.py, each pinned to the
reference): the L-level Haar w0 / w1 (``haar2d_fwd`` / ``haar2d_inv``, the
reference's ``_haar_axis_*`` primitives stopped after L levels) and the
environment irradiance E = W^{w2} L^{w2}_{top128} (``env_transfer_w2`` /
``project_environment`` / ``env_irradiance``, from ``visibility_weights`` and
``project_environment``).

The K x 3 ``csc_apply`` calls are independent; with ``workers > 1`` they run
in a fork-based process pool so the reference path uses every host core the
box gives it (each call is still the reference's own serial numba kernel).

This process never imports ``paper_2203_12339_b200`` or maps its shared
library.
"""

from __future__ import annotations

import os
import sys
import time
from pathlib import Path

import numpy as np

from . import sss_oracle as O

ROOT = Path(__file__).resolve().parents[1]
_REF = None
_POOL_STATE = {}


def import_reference(path=None):
    """Import sssrelight from baseline/_ref with the numba backend (numba
    caches go to /tmp: the installed tree stays untouched)."""
    global _REF
    if _REF is not None:
        return _REF
    path = Path(path or ROOT / "baseline" / "_ref")
    if not (path / "sssrelight").is_dir():
        raise FileNotFoundError(f"reference package not installed under {path}")
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/sss_numba_cache")
    if str(path) not in sys.path:
        sys.path.insert(0, str(path))
    import sssrelight.basisgen as basisgen
    import sssrelight.container as container
    import sssrelight.dipole as dipole
    import sssrelight.transfer as transfer
    import sssrelight.wavelets as wavelets
    from sssrelight import _accel

    _REF = {"basisgen": basisgen, "container": container, "dipole": dipole,
            "transfer": transfer, "wavelets": wavelets,
            "backend": _accel.get_kernels().__name__}
    return _REF


def _apply_task(task):
    k, c, idx, val = task
    st = _POOL_STATE  # inherited at fork: the operators, shared copy-on-write
    return k, c, st["ops"][k].apply(idx, val, st["n"])


class ReferenceFrame:
    """The reference's relight / set_material on a geometry image with the
    C3 environment light. `ops`: reference TransferOperators; `basis`: the
    reference DiffusionBasis."""

    def __init__(self, ops, basis, positions, normals, side, levels, e_keep, env_side,
                 camera, workers=1):
        self.R = import_reference()
        self.ops, self.basis = ops, basis
        self.positions = np.asarray(positions, np.float64)
        self.normals = np.asarray(normals, np.float64)
        self.side, self.levels, self.e_keep = side, levels, e_keep
        self.n = side * side
        self.camera = np.asarray(camera, np.float64)
        # frozen C3 light transfer: W^{w2} of visibility_weights
        self.w2 = O.env_transfer_w2(self.normals, env_side)
        self.workers = max(1, int(workers))
        self.vk = None
        # warm the numba kernel (JIT / cache load) outside any timing
        sp = self.R["wavelets"].compress_top_n(np.arange(self.n, dtype=np.float64), 1)
        ops[0].apply(sp.indices, sp.values, self.n)
        self.pool = None
        if self.workers > 1:
            import multiprocessing as mp

            _POOL_STATE.update(ops=self.ops, n=self.n)
            self.pool = mp.get_context("fork").Pool(self.workers)

    def close(self):
        if self.pool is not None:
            self.pool.close()
            self.pool.join()
            self.pool = None

    def relight(self, faces, material):
        """Scene.relight (runtime.py:174-187) -> (radiance, unclamped, stage ms)."""
        t = {}
        t0 = time.perf_counter()
        E = O.env_irradiance(self.w2, O.project_environment(faces, 128))
        keep = max(1, int(round(self.e_keep * self.n)))  # runtime.py:112
        spectra = []
        for c in range(3):
            coeffs = O.haar2d_fwd(E[:, c].reshape(1, self.side, self.side), self.levels).reshape(-1)
            spectra.append(self.R["wavelets"].compress_top_n(coeffs, keep))
        t1 = time.perf_counter()
        K = len(self.ops)
        vk = np.zeros((K, 3, self.n))
        tasks = [(k, c, spectra[c].indices, spectra[c].values) for k in range(K) for c in range(3)]
        if self.pool is not None:
            for k, c, out in self.pool.imap_unordered(_apply_task, tasks):
                vk[k, c] = out
        else:
            for k, c, idx, val in tasks:
                vk[k, c] = self.ops[k].apply(idx, val, self.n)
        t2 = time.perf_counter()
        self.vk = vk
        out = self.set_material(material)
        t["irradiance"] = (t1 - t0) * 1e3
        t["transfer"] = (t2 - t1) * 1e3
        t.update(out[2])
        return out[0], out[1], t, spectra

    def set_material(self, material):
        """Scene.set_material's fast path: stages 3-5 against the cached v_k."""
        sp, sa, eta = material
        t0 = time.perf_counter()
        OM = self.R["dipole"].OpticalMaterial
        s = self.R["basisgen"].project_material(
            self.basis, OM(sigma_s_prime=np.asarray(sp, np.float64),
                           sigma_a=np.asarray(sa, np.float64), eta=float(eta))).s
        summed = np.einsum("ck,kcd->cd", s, self.vk)
        t1 = time.perf_counter()
        scatter = np.empty((self.n, 3))
        for c in range(3):
            scatter[:, c] = O.haar2d_inv(summed[c].reshape(1, self.side, self.side),
                                         self.levels).reshape(-1)
        view = self.camera[None, :] - self.positions
        view /= np.linalg.norm(view, axis=1, keepdims=True)
        cos = np.clip(np.einsum("ij,ij->i", self.normals, view), 0.0, 1.0)
        ft = self.R["dipole"].fresnel_transmittance(float(eta), cos)
        unclamped = scatter * (ft / np.pi)[:, None]
        t2 = time.perf_counter()
        return np.maximum(unclamped, 0.0), unclamped, {"weighting": (t1 - t0) * 1e3,
                                                        "inverse_wavelet": (t2 - t1) * 1e3}


def load_reference_container(path):
    """The reference's own PRTS1 loader (container.py:156-235)."""
    R = import_reference()
    return R["container"].load_container(str(path))


def time_sequence(frame: ReferenceFrame, faces, mats, warmup, steps, material0):
    """The bench sequence on the reference: per step a relight with the
    step's cubemap; on edit steps a set_material too. Returns per-step seconds
    (after `warmup` untimed steps)."""
    material = material0
    times = []
    for f in range(warmup + steps):
        t0 = time.perf_counter()
        frame.relight(faces[f], material)
        if f in mats:
            material = mats[f]
            frame.set_material(material)
        dt = time.perf_counter() - t0
        if f >= warmup:
            times.append(dt)
    return times
