"""CPU-only checks: host logic, index maps, the C ABI library's exports."""

import ctypes
import re
from pathlib import Path

import numpy as np
import torch
import pytest

from oracle import sss_oracle as O
from paper_2203_12339_b200 import config as C
from paper_2203_12339_b200 import lighting as LT
from paper_2203_12339_b200.geometry import make_geometry_image
from paper_2203_12339_b200.transfer import (DeviceTransfer, TransferOperator,
                                            flat_to_tile_major, tile_major_to_flat)

ROOT = Path(__file__).resolve().parents[1]


@pytest.mark.parametrize("side,L", [(8, 1), (16, 2), (32, 2), (64, 3), (32, 5)])
def test_tile_major_map_matches_oracle(side, L):
    flat = np.arange(side * side)
    tm = flat_to_tile_major(flat, side, L)
    assert np.array_equal(np.sort(tm), flat)  # bijection
    T = 1 << L
    for f in flat[:: max(1, side * side // 257)]:
        tr, tc = O.coeff_tile(f // side, f % side, side, L)
        assert tm[f] // (T * T) == tr * (side // T) + tc
    perm = tile_major_to_flat(side, L)
    assert np.array_equal(flat_to_tile_major(perm, side, L), flat)


def test_tile_local_layout_is_tile_haar():
    """Gathering a tile's coefficients in tile-major order gives the tile's
    own full-pyramid Haar (the fused epilogue's premise)."""
    side, L = 32, 3
    T = 1 << L
    x = np.random.default_rng(3).standard_normal((side, side))
    h = O.haar2d_fwd(x[None], L)[0].reshape(-1)
    perm = tile_major_to_flat(side, L)
    tiles = h[perm].reshape(-1, T, T)
    tr, tc = 2, 1
    want = O.haar2d_fwd(x[None, tr * T:(tr + 1) * T, tc * T:(tc + 1) * T])[0]
    assert np.array_equal(tiles[tr * (side // T) + tc], want)


def test_operator_layout_round_trip():
    rng = np.random.default_rng(5)
    side, L, K = 16, 2, 3
    n = side * side
    ops = []
    for _ in range(K):
        cols = np.sort(rng.choice(n, 40, replace=False)).astype(np.uint32)
        counts = rng.integers(0, 12, cols.size)
        colptr = np.zeros(cols.size + 1, np.int64)
        colptr[1:] = np.cumsum(counts)
        rowidx = np.concatenate([np.sort(rng.choice(n, c, replace=False)) for c in counts]).astype(np.uint32)
        vals = rng.standard_normal(rowidx.size).astype(np.float32).astype(np.float64)
        ops.append(TransferOperator(cols, colptr, rowidx, vals))
    dt = DeviceTransfer.from_reference(ops, side, L, device="cpu")
    back = dt.to_reference()
    for a, b in zip(ops, back):
        keep = np.diff(a.colptr) > 0
        assert np.array_equal(a.cols[keep], b.cols)
        assert np.array_equal(a.rowidx, b.rowidx)
        assert np.array_equal(a.vals, b.vals)
    # dense product equivalence (the frame layout computes the same thing)
    x = rng.standard_normal(n)
    perm = tile_major_to_flat(side, L)
    x_tm = x[perm]  # operator columns are tile-major ids
    rp = dt.rowptr.numpy()
    cols = dt.cols.numpy().view(np.uint32)
    vals = dt.vals.numpy().astype(np.float64)
    for k, op in enumerate(ops):
        want = O.csc_apply(op.cols, op.colptr, op.rowidx, op.vals, np.arange(n, dtype=np.uint32), x, n)
        got = np.zeros(n)
        for r in range(n):
            sl = slice(rp[k, r], rp[k, r + 1])
            assert np.all(np.diff(cols[sl].astype(np.int64)) > 0)  # ascending within a row
            got[perm[r]] = np.dot(vals[sl], x_tm[cols[sl]])
        assert np.allclose(got, want, rtol=1e-12, atol=1e-12)


def _random_device_transfer(rng, side, L, K, per_col):
    n = side * side
    ops = []
    shared = np.sort(rng.choice(n, per_col, replace=False))  # overlapping supports across k
    for _ in range(K):
        cols = np.sort(rng.choice(n, 60, replace=False)).astype(np.uint32)
        colptr = np.zeros(cols.size + 1, np.int64)
        rows = []
        for i in range(cols.size):
            pick = np.unique(np.concatenate([rng.choice(shared, per_col // 2, replace=False),
                                             rng.choice(n, rng.integers(0, per_col), replace=False)]))
            rows.append(pick)
            colptr[i + 1] = colptr[i] + pick.size
        rowidx = np.concatenate(rows).astype(np.uint32)
        vals = rng.standard_normal(rowidx.size).astype(np.float32).astype(np.float64)
        ops.append(TransferOperator(cols, colptr, rowidx, vals))
    return DeviceTransfer.from_reference(ops, side, L, device="cpu")


def _csr_vk(dt, x_tm):
    rp = dt.rowptr.numpy()
    cols = dt.cols.numpy().view(np.uint32)
    vals = dt.vals.numpy().astype(np.float64)
    vk = np.zeros((dt.K, 3, dt.n))
    for k in range(dt.K):
        for r in range(dt.n):
            sl = slice(rp[k, r], rp[k, r + 1])
            vk[k, :, r] = vals[sl] @ x_tm[cols[sl]]
    return vk


def test_library_exports_every_header_symbol():
    from paper_2203_12339_b200 import _lib, build

    build.build()
    lib = _lib.load(require_cuda=False)
    header = (ROOT / "include" / "sss_b200.h").read_text()
    declared = set(re.findall(r"^\s*(?:int|const char\*)\s+(sss_\w+)\(", header, re.M))
    assert declared == set(_lib.exported_symbols())
    for name in declared:
        assert isinstance(getattr(lib, name), ctypes._CFuncPtr)
    assert lib.sss_version() == 1


def test_library_rejects_bad_arguments_without_gpu():
    from paper_2203_12339_b200 import _lib

    lib = _lib.load(require_cuda=False)
    rc = lib.sss_haar2d(None, None, 1, 12, 2, 0, None)  # side not a power of two
    assert rc == -1 and b"power of two" in lib.sss_last_error()
    rc = lib.sss_select_topn(None, 1, 16, 4, None, None, None, None, None)
    assert rc == -1


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
def test_product_path_fails_loudly_without_gpu_or_library(monkeypatch, tmp_path):
    """No CPU fallback: without a GPU the API raises (even after a CPU-side
    load of the library for symbol checks), and a missing .so raises too."""
    from paper_2203_12339_b200 import _lib
    from paper_2203_12339_b200.runtime import Scene

    _lib.load(require_cuda=False)
    with pytest.raises(_lib.SSSError, match="CUDA device required"):
        _lib.load()
    with pytest.raises(_lib.SSSError, match="CUDA device required"):
        Scene(None, None, None, None, None)
    monkeypatch.setattr(_lib, "_lib", None)
    monkeypatch.setattr(_lib, "_SO", tmp_path / "missing.so")
    with pytest.raises(_lib.SSSError, match="no CPU fallback"):
        _lib.load(require_cuda=False)


def test_geometry_image_properties():
    g = make_geometry_image(32)
    assert g.positions.dtype == np.float32 and g.positions.shape == (1024, 3)
    assert np.allclose(np.linalg.norm(g.normals, axis=1), 1.0, atol=1e-6)
    r = np.linalg.norm(g.positions, axis=1)
    assert 0.6 * 10 < r.min() and r.max() < 1.4 * 10
    assert np.all(g.area > 0) and abs(g.area.sum() / (4 * np.pi * 100) - 1) < 0.1
    # determinism
    assert np.array_equal(make_geometry_image(32).positions, g.positions)


def test_sh_basis_orthonormal_and_transfer_closed_form():
    s = 96
    d = LT.face_directions(s).reshape(-1, 3)
    w = LT.face_solid_angles(s).reshape(-1)
    Y = LT.sh_eval(d, 5)
    G = (Y * w[:, None]).T @ Y
    assert np.abs(G - np.eye(25)).max() < 1e-3
    g = make_geometry_image(16)
    n = g.normals.astype(np.float64)
    Wq = O.visibility_weights(n, s)  # reference-anchored quadrature (lighting.py:318-329)
    Tq = Wq @ Y
    Ta = LT.sh_transfer(n, 5)
    assert np.abs(Tq - Ta).max() < 2e-4 * np.abs(Ta).max()


def test_sh_rotation_exact():
    rng = np.random.default_rng(9)
    R = LT.random_rotation(rng)
    assert np.allclose(R @ R.T, np.eye(3), atol=1e-12) and np.linalg.det(R) > 0
    c = LT.random_sh_light(5, 4)
    cr = LT.rotate_sh(c, R)
    w = rng.standard_normal((50, 3))
    w /= np.linalg.norm(w, axis=1, keepdims=True)
    assert np.abs(LT.sh_eval(w, 5) @ cr - LT.sh_eval(w @ R, 5) @ c).max() < 1e-12


def test_environment_rotation_and_tables():
    env = LT.Environment(side=16, seed=3)
    f0, f90 = env.faces(0.0), env.faces(90.0)
    assert f0.shape == (6, 16, 16, 3) and np.all(f0 > 0)
    assert f0.max() > 40  # lobes present
    assert not np.array_equal(f0, f90)
    assert np.array_equal(LT.face_directions(8), O.face_directions(8))
    assert np.array_equal(LT.face_solid_angles(8), O.face_solid_angles(8))


def test_product_basis_matches_golden(golden):
    from paper_2203_12339_b200.basis import build_basis

    g = golden("basis")
    b = build_basis(4, (4, 4))
    assert np.array_equal(b.r_nodes, g["r_nodes"])
    assert np.abs(b.bases - g["4x4_K4_bases"]).max() <= 1e-9 * np.abs(g["4x4_K4_bases"]).max()


def test_configs_frozen():
    assert C.C1.n == 1024 and C.C2.n == 16384 and C.C3.n == 65536
    assert C.C1.n_materials == 16 and C.C2.n_materials == 32 and C.C5.n_materials == 64
    assert C.STEP2_FRACTION == 0.95 and C.E_KEEP == 0.25


def test_kfr_layout_reproduces_csr_product():
    """The K-fused row-chunk stream of sss_transfer_kfr (layout.kfr_layout),
    decoded the way the kernel reads it (compacted words per step, term
    planes, partial sums of multi-chunk rows), computes the per-term CSR
    product; every coefficient appears exactly once."""
    from paper_2203_12339_b200.layout import kfr_layout, kfr_reference_apply

    rng = np.random.default_rng(12)
    dt = _random_device_transfer(rng, 32, 2, 5, 24)
    x_tm = rng.standard_normal((dt.n, 3))
    want = _csr_vk(dt, x_tm)
    for chunk, steps in ((512, 4), (8, 4), (64, 8)):  # 8: rows span several chunks
        lay = kfr_layout(dt, chunk=chunk, steps_per_batch=steps)
        assert lay.stats["entries"] == dt.nnz
        assert int((lay.lane_len.long() & 0xFFFFFFFF).sum()) == lay.stats["pairs"]
        if chunk == 8:
            assert lay.n_partials > 0
        bo = lay.batch_off.long() & 0xFFFFFFFF
        assert torch.all(bo % 16 == 0) and int(bo[-1]) <= 4 * lay.stream.numel()
        got = kfr_reference_apply(lay, torch.as_tensor(x_tm.T.copy())).numpy()
        assert np.allclose(got, want, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("col16", [True, False])
def test_flat16_layout_reproduces_csr_product(col16):
    """The flat16 stream (layout.flat16_layout): (row, k) segments padded to 16
    entries and lane-interleaved, head bits at segment starts."""
    from paper_2203_12339_b200.layout import flat16_layout

    rng = np.random.default_rng(13)
    dt = _random_device_transfer(rng, 32, 2, 5, 24)
    x_tm = rng.standard_normal((dt.n, 3))
    want = _csr_vk(dt, x_tm)
    pcols, pvals, ne, heads, hpre, rowk, wbeg, W, st = flat16_layout(dt, warps_per_sm=1, col16=col16)
    cols = pcols.numpy().astype(np.int64) & (0xFFFF if col16 else 0xFFFFFFFF)
    vals = pvals.numpy().astype(np.float64)
    hb = heads.numpy().view(np.uint32)
    rowk = rowk.numpy()
    ng = ne // 16
    starts = [g for g in range(ng) if (hb[g // 32] >> (g % 32)) & 1]
    assert len(starts) == rowk.size and starts[0] == 0
    xpad = np.vstack([x_tm, np.zeros((1, 3))])
    got = np.zeros_like(want)
    for i, g0 in enumerate(starts):
        g1 = starts[i + 1] if i + 1 < len(starts) else ng
        sl = slice(g0 * 16, g1 * 16)
        r, k = rowk[i] >> 4, rowk[i] & 15
        got[k, :, r] += vals[sl] @ xpad[cols[sl]]
    assert np.allclose(got, want, rtol=1e-12, atol=1e-12)


def _bvh_any_hit_py(bvh, o, d, tmax):
    """The GPU traversal restated (stack, slab AABB test, reference triangle
    test in the numba operation order): test-side check of the BVH build."""
    stack = [0]
    while stack:
        nd = stack.pop()
        tn, tf = 0.0, tmax
        ok = True
        for ax in range(3):
            lo, hi = bvh.node_min[nd, ax], bvh.node_max[nd, ax]
            if d[ax] == 0.0:
                if o[ax] < lo or o[ax] > hi:
                    ok = False
                    break
            else:
                inv = 1.0 / d[ax]
                ta, tb = (lo - o[ax]) * inv, (hi - o[ax]) * inv
                if ta > tb:
                    ta, tb = tb, ta
                tn, tf = max(tn, ta), min(tf, tb)
                if tn > tf:
                    ok = False
                    break
        if not ok:
            continue
        c = bvh.node_count[nd]
        if c > 0:
            s = bvh.node_start[nd]
            if O.tri_any_hit(np.repeat(o[None], c, 0), np.repeat(d[None], c, 0), np.full(c, tmax),
                             bvh.v0[s:s + c], bvh.e1[s:s + c], bvh.e2[s:s + c]).any():
                return True
        else:
            stack += [bvh.node_left[nd], bvh.node_right[nd]]
    return False


def test_bvh_any_hit_matches_reference_rays(golden):
    from paper_2203_12339_b200.shadows import build_bvh

    g = golden("direct")
    bvh = build_bvh(g["positions"], g["triangles"])
    assert bvh.ray_offset == float(g["ray_offset"])
    got = np.array([_bvh_any_hit_py(bvh, o, d, t)
                    for o, d, t in zip(g["ray_o"], g["ray_d"], g["ray_t"])])
    assert np.array_equal(got, g["hits"])
    # structure: leaves partition the triangles
    leaves = bvh.node_count > 0
    assert bvh.node_count[leaves].sum() == g["triangles"].shape[0]
    assert np.all(bvh.node_count <= 4)


def test_bvh_packed_records(golden):
    """The GPU node / triangle records carry the BVH fields bit for bit."""
    from paper_2203_12339_b200.shadows import LightRig, PointLight, SphereLight, build_bvh

    g = golden("direct")
    bvh = build_bvh(g["positions"], g["triangles"])
    nodes, tris = bvh.packed()
    assert nodes.shape == (bvh.node_min.shape[0], 8) and tris.shape == (bvh.v0.shape[0], 10)
    assert np.array_equal(nodes[:, :3], bvh.node_min) and np.array_equal(nodes[:, 3:6], bvh.node_max)
    ints = nodes.view(np.int32)
    for col, a in zip((12, 13, 14, 15), (bvh.node_left, bvh.node_right, bvh.node_start,
                                         bvh.node_count)):
        assert np.array_equal(ints[:, col], a)
    assert np.array_equal(tris[:, 0:3], bvh.v0) and np.array_equal(tris[:, 6:9], bvh.e2)
    rig = LightRig(lights=(SphereLight(center=[0, 0, 5], radius=1, radiance=1),
                           PointLight(position=[1, 2, 3], intensity=4)))
    assert rig.kinds().tolist() == [2, 0] and rig.kinds().dtype == np.int32
