"""GPU parity for visibility precompute + ambient folding (SURVEY §8f row 3,
transfer.py:368-451, runtime.py:146-149) against the reference's own output
(tests/golden/fold.npz) and the oracle.

Bars: visibility bitwise (except directions within 1e-9 of the horizon,
where the reference's BLAS `normals @ dirs.T` and the device's ordered dot
product may round the sign of cos differently); folded kept sets identical
to the oracle on the same f32 operator values wherever the energy cut is
not within 1e-9 of a tie; folded values within one f32 rounding; the
folded ambient v_k bitwise against the oracle's serial csc_apply on the
stored values.
"""

from types import SimpleNamespace

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import sss_oracle as O  # noqa: E402


@pytest.fixture(scope="module")
def lib():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    from paper_2203_12339_b200 import _lib, build

    build.build()
    return _lib.load()


def _geom(d):
    return SimpleNamespace(positions=d["positions"].astype(np.float32),
                           normals=d["normals"].astype(np.float32), side=int(d["side"]))


def _ops(g, tag, K=4):
    return [O.Operator(g[f"{tag}{k}_cols"], g[f"{tag}{k}_colptr"], g[f"{tag}{k}_rowidx"],
                       g[f"{tag}{k}_vals"], float(g[f"{tag}{k}_e"][0]), float(g[f"{tag}{k}_e"][1]),
                       int(g[f"{tag}{k}_e"][2])) for k in range(K)]


def _device_transfer(ops, side):
    from paper_2203_12339_b200.transfer import DeviceTransfer, TransferOperator

    L = int(np.log2(side))
    refs = [TransferOperator(cols=o.cols, colptr=o.colptr, rowidx=o.rowidx, vals=o.vals,
                             kept_energy=o.kept_energy, total_energy=o.total_energy,
                             step1_entries=o.step1_entries) for o in ops]
    return DeviceTransfer.from_reference(refs, side, L)


def _union(spectra):
    idx = np.unique(np.concatenate([s.indices for s in spectra])).astype(np.uint32)
    lc = np.zeros((idx.size, 3))
    for c, s in enumerate(spectra):
        lc[np.searchsorted(idx, s.indices), c] = s.values
    dev = lambda a, dt: torch.as_tensor(np.ascontiguousarray(a, dt), device="cuda")
    return (dev(idx.view(np.int32), np.int32), dev(lc, np.float64),
            dev(np.array([idx.size]), np.int32))


def test_visibility_vs_reference(lib, golden):
    from paper_2203_12339_b200.folding import precompute_visibility

    g, d = golden("fold"), golden("direct")
    fs = int(g["face_side"])
    vis = precompute_visibility(_geom(d), face_side=fs)
    got = vis.matrix()
    want = g["vis"].astype(np.float64)
    cos = d["normals"] @ O.face_directions(fs).reshape(-1, 3).T
    differ = got != want
    assert not np.any(differ & (np.abs(cos) > 1e-9)), np.argwhere(differ)[:5]
    assert 0.2 < got.mean() < 0.8


def test_fold_vs_oracle_and_reference(lib, golden):
    from paper_2203_12339_b200.folding import DeviceVisibility, fold_visibility

    g, d = golden("fold"), golden("direct")
    side, fs, eta, frac = int(g["side"]), int(g["face_side"]), float(g["eta"]), float(g["fraction"])
    ops = [O.round_trip_f32(o) for o in _ops(g, "op")]
    dt = _device_transfer(ops, side)
    vis = DeviceVisibility(vis=torch.as_tensor(np.ascontiguousarray(g["vis"].T), device="cuda"),
                           face_side=fs)
    folded = fold_visibility(dt, vis, _geom(d), eta, frac)
    got = folded.to_reference()
    want, dense = O.fold_visibility(ops, g["vis"].astype(np.float64), d["normals"], side, fs, eta,
                                    frac)
    n_cols = n_skipped = 0
    for k in range(4):
        gk, wk = got[k], want[k]
        assert np.array_equal(gk.cols, wk.cols)
        assert gk.step1_entries == wk.step1_entries
        assert gk.kept_energy == pytest.approx(wk.kept_energy, rel=1e-9)
        assert gk.total_energy == pytest.approx(wk.total_energy, rel=1e-9)
        for ci, e in enumerate(wk.cols):
            n_cols += 1
            gs = slice(gk.colptr[ci], gk.colptr[ci + 1])
            ws = slice(wk.colptr[ci], wk.colptr[ci + 1])
            if not np.array_equal(gk.rowidx[gs], wk.rowidx[ws]):
                assert O.energy_select_margin(dense[k][:, e], frac) < 1e-9, (k, e)
                n_skipped += 1
                continue
            wv = wk.vals[ws].astype(np.float32).astype(np.float64)
            assert np.allclose(gk.vals[gs], wv, rtol=2.0 ** -22, atol=0.0), (k, e)
    assert n_skipped <= max(1, n_cols // 100)
    # against the reference's fold on its f64 operator values: same column
    # sets, kept sets equal in at least 99 % of the columns
    ref = _ops(g, "fold")
    same = sum(np.array_equal(got[k].rowidx[got[k].colptr[i]:got[k].colptr[i + 1]],
                              ref[k].rowidx[ref[k].colptr[i]:ref[k].colptr[i + 1]])
               for k in range(4) for i in range(ref[k].cols.size))
    assert all(np.array_equal(got[k].cols, ref[k].cols) for k in range(4))
    assert same >= 0.99 * sum(r.cols.size for r in ref)


def test_fold_apply_bitwise(lib, golden):
    from paper_2203_12339_b200.folding import DeviceVisibility, fold_apply, fold_visibility
    from paper_2203_12339_b200.transfer import tile_major_to_flat

    g, d = golden("fold"), golden("direct")
    side, fs = int(g["side"]), int(g["face_side"])
    n = side * side
    ops = [O.round_trip_f32(o) for o in _ops(g, "op")]
    vis = DeviceVisibility(vis=torch.as_tensor(np.ascontiguousarray(g["vis"].T), device="cuda"),
                           face_side=fs)
    folded = fold_visibility(_device_transfer(ops, side), vis, _geom(d), float(g["eta"]),
                             float(g["fraction"]))
    spectra = [O.Spectrum(g[f"env_idx{c}"], g[f"env_val{c}"], 6 * fs * fs, 0.0, 0.0)
               for c in range(3)]
    base = np.random.default_rng(3).standard_normal((4, 3, n))
    perm = tile_major_to_flat(side, int(np.log2(side)))
    amb = O.ambient_vk(folded.to_reference(), spectra, n)
    for layout in ("rows", "csc"):  # the row-major (default) and CSC kernels
        vk = torch.as_tensor(base, device="cuda")  # tile-major rows
        fold_apply(folded, *_union(spectra), vk, layout=layout)
        torch.cuda.synchronize()
        got = vk.cpu().numpy()[:, :, np.argsort(perm)]  # -> flat rows
        assert np.array_equal(got, base[:, :, np.argsort(perm)] + amb), layout
    # the reference's folded ambient v_k (its own f64 fold of f64 operators)
    assert np.abs(amb - g["vk"]).max() <= 1e-5 * np.abs(g["vk"]).max()


def test_zero_visibility_folds_to_zero(lib, golden):
    from paper_2203_12339_b200.folding import DeviceVisibility, fold_visibility

    g, d = golden("fold"), golden("direct")
    side, fs = int(g["side"]), int(g["face_side"])
    vis = DeviceVisibility(vis=torch.zeros((6 * fs * fs, side * side), dtype=torch.uint8,
                                           device="cuda"), face_side=fs)
    folded = fold_visibility(_device_transfer(_ops(g, "op"), side), vis, _geom(d), 1.3)
    assert all(o.cols.size == 0 and o.rowidx.size == 0 for o in folded.to_reference())
    with pytest.raises(ValueError):
        fold_visibility(_device_transfer(_ops(g, "op"), side),
                        DeviceVisibility(vis=vis.vis[:, :3], face_side=fs), _geom(d), 1.3)
