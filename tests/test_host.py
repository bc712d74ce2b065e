"""CPU-only checks: host logic, index maps, the C ABI library's exports."""

import ctypes
import re
from pathlib import Path

import numpy as np
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
