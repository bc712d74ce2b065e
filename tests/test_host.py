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
    bo = dt.bandoff.numpy()
    for k, op in enumerate(ops):
        want = O.csc_apply(op.cols, op.colptr, op.rowidx, op.vals, np.arange(n, dtype=np.uint32), x, n)
        got = np.zeros(n)
        for r in range(n):
            sl = slice(rp[k, r], rp[k, r + 1])
            assert np.all(np.diff(cols[sl].astype(np.int64)) > 0)  # ascending within a row
            got[perm[r]] = np.dot(vals[sl], x_tm[cols[sl]])
            # band offsets partition the row by column band
            for b in range(dt.n_bands):
                seg = cols[rp[k, r] + bo[k, r, b]: rp[k, r] + bo[k, r, b + 1]]
                assert np.all(seg // dt.band_width == b)
            assert bo[k, r, dt.n_bands] == rp[k, r + 1] - rp[k, r]
        assert np.allclose(got, want, rtol=1e-12, atol=1e-12)
    # rowperm: a permutation within each unit, longest rows first
    R = dt.unit_tiles * (1 << L) ** 2
    pr = dt.rowperm.numpy()
    assert np.array_equal(np.sort(pr), np.arange(n))
    assert np.all(pr // R == np.arange(n) // R)


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


def test_kstep_layout_reproduces_csr_product():
    """The mask-sorted K-fused warp-step layout (sss_transfer_kstep) computes
    the same v_k as the per-term CSR: emulate the kernel over the layout."""
    from paper_2203_12339_b200.runtime import kstep_layout

    rng = np.random.default_rng(12)
    dt = _random_device_transfer(rng, 32, 2, 5, 24)
    x_tm = rng.standard_normal((dt.n, 3))
    want = _csr_vk(dt, x_tm)
    cols, vals, steps, wbeg, W, stats = kstep_layout(dt, warps_per_sm=1)
    cols = cols.numpy().view(np.uint32)
    vals = vals.numpy().astype(np.float64)
    steps = steps.numpy().view(np.uint32)
    wbeg = wbeg.numpy()
    assert wbeg[0] == 0 and wbeg[-1] == steps.shape[0] and np.all(np.diff(wbeg) >= 0)
    assert stats["pairs"] <= int(dt.rowptr[:, -1].max() - dt.rowptr[0, 0])
    got = np.zeros_like(want)
    rows_seen = []
    for s in range(steps.shape[0]):
        p0, v0, row, info = (int(v) for v in steps[s])
        mask, cnt, end = info & 0xFF, (info >> 8) & 0xFF, (info >> 16) & 1
        assert 1 <= cnt <= 32 and v0 % 32 == 0
        xs = x_tm[cols[p0:p0 + cnt]]
        j = 0
        for k in range(8):
            if mask >> k & 1:
                v = vals[v0 + 32 * j: v0 + 32 * j + 32]
                assert np.all(v[cnt:] == 0)
                got[k, :, row] += v[:cnt] @ xs
                j += 1
        if end:
            rows_seen.append(row)
    assert len(rows_seen) == len(set(rows_seen))
    assert np.allclose(got, want, rtol=1e-12, atol=1e-12)


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


def test_kstream_blobs_reproduce_csr_product():
    """sss_transfer_kstream's per-step blobs [32 columns | popc x 32 values]
    carry the same v_k as the per-term CSR (kernel emulated on the host)."""
    from paper_2203_12339_b200.runtime import kstream_layout

    rng = np.random.default_rng(13)
    dt = _random_device_transfer(rng, 32, 2, 6, 20)
    x_tm = rng.standard_normal((dt.n, 3))
    want = _csr_vk(dt, x_tm)
    blob, recs, wbeg, W, stats = kstream_layout(dt, warps_per_sm=1)
    blob = blob.numpy()
    recs = recs.numpy().view(np.uint32)
    wbeg = wbeg.numpy()
    assert wbeg[0] == 0 and wbeg[-1] == recs.shape[0] and W % 8 == 0
    bcols = blob.view(np.uint32)
    bvals = blob.view(np.float32).astype(np.float64)
    got = np.zeros_like(want)
    for s in range(recs.shape[0]):
        off, row, info = int(recs[s, 0]) * 4, int(recs[s, 1]), int(recs[s, 2])
        mask, cnt = info & 0xFF, (info >> 8) & 0xFF
        assert np.all(bcols[off + cnt: off + 32] == 0)
        xs = x_tm[bcols[off: off + 32]]
        j = 0
        for k in range(8):
            if mask >> k & 1:
                got[k, :, row] += bvals[off + 32 + 32 * j: off + 64 + 32 * j] @ xs
                j += 1
        if s + 1 < recs.shape[0]:
            assert int(recs[s + 1, 0]) * 4 == off + 32 * (1 + j)  # contiguous blobs
    assert np.allclose(got, want, rtol=1e-12, atol=1e-12)


def test_kgroup_layout_reproduces_csr_product():
    """sss_transfer_kgroup's K-packed, 32-padded row pieces carry the same v_k
    as the per-term CSR (kernel emulated on the host, unkept columns skipped)."""
    from paper_2203_12339_b200.runtime import kgroup_layout

    rng = np.random.default_rng(14)
    dt = _random_device_transfer(rng, 32, 2, 7, 40)
    x_tm = rng.standard_normal((dt.n, 3))
    x_tm[rng.random(dt.n) < 0.6] = 0.0  # unkept columns
    want = _csr_vk(dt, x_tm)
    meta, vals, pieces, wbeg, W, stats = kgroup_layout(dt, warps_per_sm=1, split=64)
    assert stats["pieces"] > dt.n - np.count_nonzero(
        (dt.rowptr[:, 1:] - dt.rowptr[:, :-1]).sum(0).numpy() == 0)  # some rows split
    meta = meta.numpy().view(np.uint32)
    vals = vals.numpy().astype(np.float64)
    pieces = pieces.numpy().view(np.uint32)
    wbeg = wbeg.numpy()
    assert wbeg[0] == 0 and wbeg[-1] == pieces.shape[0] and np.all(np.diff(wbeg) >= 0)
    kept = np.any(x_tm != 0, axis=1)
    got = np.zeros_like(want)
    for p0, npair, v0, row in pieces:
        assert p0 % 32 == 0 and npair % 32 == 0 and 0 < npair <= 64
        off = v0
        for m in meta[p0:p0 + npair]:
            mask, col = int(m) >> 24, int(m) & 0xFFFFFF
            for k in range(8):
                if mask >> k & 1:
                    if kept[col]:
                        got[k, :, row] += vals[off] * x_tm[col]
                    off += 1
    assert np.allclose(got, want, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("group,perm", [(4, False), (8, False), (8, True)])
def test_flat_stream_layout_reproduces_csr_product(group, perm):
    """sss_transfer_flat's head-flag bitmap / segment prefix over the padded
    operator copy recover every segment's (row, k): emulate the segmented
    warp-stream on the host, including warp ranges that cut segments."""
    from paper_2203_12339_b200.runtime import flat_layout

    rng = np.random.default_rng(15)
    dt = _random_device_transfer(rng, 32, 2, 5, 30)
    x_tm = rng.standard_normal((dt.n, 3))
    want = _csr_vk(dt, x_tm)
    from paper_2203_12339_b200.runtime import block_column_order

    order = None
    if perm:
        new_of, tm_of = block_column_order(32, 2)
        assert np.array_equal(np.sort(new_of), np.arange(dt.n))
        order = new_of
        x_tm = x_tm[tm_of]  # the kernel reads x in the permuted column order
    pcols, pvals, ne, heads, hpre, rowk, wbeg, W, stats = flat_layout(dt, warps_per_sm=1,
                                                                       group=group, col_order=order)
    c4 = pcols.numpy().view(np.uint32).reshape(-1, group)
    v4 = pvals.numpy().astype(np.float64).reshape(-1, group)
    heads = heads.numpy().view(np.uint32)
    hpre = hpre.numpy().view(np.uint32)
    rowk = rowk.numpy().view(np.uint32)
    wbeg = wbeg.numpy()
    assert ne == c4.size and wbeg[0] == 0 and wbeg[-1] == heads.size
    got = np.zeros_like(want)
    n4 = c4.shape[0]
    for w in range(W):
        for i in range(wbeg[w], wbeg[w + 1]):
            for lane in range(32):
                q = 32 * i + lane
                if q >= n4:
                    continue
                hm = int(heads[i]) & ((2 << lane) - 1)
                pid = int(hpre[i]) + bin(hm).count("1") - 1
                rk = int(rowk[pid])
                got[rk & 15, :, rk >> 4] += v4[q] @ x_tm[c4[q]]
    assert np.allclose(got, want, rtol=1e-12, atol=1e-12)


def test_regional_layout_reproduces_csr_product():
    """v19 regional layout: region-local slots map back to columns through
    each region's union list; regions span whole 256-entry iterations; the
    head-flag stream gives every segment's (row, k) (host emulation)."""
    from paper_2203_12339_b200.runtime import regional_layout

    rng = np.random.default_rng(19)
    dt = _random_device_transfer(rng, 32, 2, 4, 30)
    x_tm = rng.standard_normal((dt.n, 3))
    x_tm[rng.random(dt.n) < 0.5] = 0.0
    want = _csr_vk(dt, x_tm)
    R = regional_layout(dt)
    c8 = R["pcols"].numpy().view(np.uint32).reshape(-1, 8)
    v8 = R["pvals"].numpy().astype(np.float64).reshape(-1, 8)
    heads = R["heads"].numpy().view(np.uint32)
    hpre = R["hpre"].numpy().view(np.uint32)
    rowk = R["rowk"].numpy().view(np.uint32)
    ucols = R["ucols"].numpy().view(np.uint32)
    uoff = R["uoff"].numpy()
    rit = R["rit"].numpy()
    T2 = 16
    assert rit[-1] * 32 == c8.shape[0] or rit[-1] * 32 >= c8.shape[0] - 31
    got = np.zeros_like(want)
    for r in range(R["n_regions"]):
        u = ucols[uoff[r]:uoff[r + 1]]
        assert np.all(np.diff(u.astype(np.int64)) > 0)
        for i in range(rit[r], rit[r + 1]):
            for lane in range(32):
                q = 32 * i + lane
                if q >= c8.shape[0]:
                    continue
                hm = int(heads[i]) & ((2 << lane) - 1)
                pid = int(hpre[i]) + bin(hm).count("1") - 1
                rk = int(rowk[pid])
                assert (rk >> 4) // T2 == r  # the segment belongs to this region
                got[rk & 15, :, rk >> 4] += v8[q] @ x_tm[u[c8[q]]]
    assert np.allclose(got, want, rtol=1e-12, atol=1e-12)


def test_k8_dense_pairs_layout_reproduces_csr_product():
    """v20 dense K-fused pairs: one lane per (row, column) pair with its K
    values at slots 0..K-1; padding pairs carry column N (host emulation)."""
    from paper_2203_12339_b200.runtime import k8_layout

    rng = np.random.default_rng(20)
    dt = _random_device_transfer(rng, 32, 2, 6, 30)
    x_tm = rng.standard_normal((dt.n, 3))
    x_tm[rng.random(dt.n) < 0.5] = 0.0
    want = _csr_vk(dt, x_tm)
    cols, vals, pieces, wbeg, W, stats = k8_layout(dt, warps_per_sm=1, split=64)
    cols = cols.numpy().view(np.uint32)
    vals = vals.numpy().astype(np.float64)
    pieces = pieces.numpy()
    wbeg = wbeg.numpy()
    assert wbeg[0] == 0 and wbeg[-1] == pieces.shape[0]
    got = np.zeros_like(want)
    for p0, pn, row, _ in pieces:
        assert p0 % 32 == 0 and pn % 32 == 0 and 0 < pn <= 64
        for p in range(p0, p0 + pn):
            c = int(cols[p])
            if c >= dt.n:
                assert np.all(vals[p] == 0)
                continue
            for k in range(dt.K):
                got[k, :, row] += vals[p, k] * x_tm[c]
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
