"""The reference arm (bench.py --impl reference / cpu_baseline): the frame
composed from the reference's own code (baseline/_ref sssrelight, numba)
equals the oracle's frame, serially and over a process pool. CPU only."""

import numpy as np
import pytest

from oracle import sss_oracle as O


@pytest.fixture(scope="module")
def small():
    from oracle.reference_frame import import_reference

    try:
        R = import_reference()
    except FileNotFoundError:
        pytest.skip("reference not installed under baseline/_ref")
    from paper_2203_12339_b200 import lighting as LT
    from paper_2203_12339_b200.basis import build_basis
    from paper_2203_12339_b200.geometry import make_geometry_image

    side, L, keep, frac = 16, 2, 0.10, 0.95
    g = make_geometry_image(side)
    b = build_basis(4, (4, 4))
    ops = O.precompute_compressed(g.positions.astype(np.float64), g.area.astype(np.float64), side,
                                  b.r_nodes, b.bases, keep, frac, levels=L, w1="haar")
    ops = [O.round_trip_f32(o) for o in ops]
    rops = [R["transfer"].TransferOperator(cols=o.cols, colptr=o.colptr, rowidx=o.rowidx,
                                           vals=o.vals, kept_energy=o.kept_energy,
                                           total_energy=o.total_energy,
                                           step1_entries=o.step1_entries) for o in ops]
    rb = R["basisgen"].DiffusionBasis(r_nodes=b.r_nodes, bases=b.bases,
                                      singular_values=b.singular_values, eta=b.eta, g=b.g,
                                      sigma_box=tuple(b.sigma_box))
    env = LT.Environment(side=8, seed=3)
    return side, L, g, b, ops, rops, rb, env


@pytest.mark.parametrize("workers", [1, 2])
def test_reference_frame_equals_oracle_frame(small, workers):
    from oracle.reference_frame import ReferenceFrame

    side, L, g, b, ops, rops, rb, env = small
    cam = np.array([0.0, 0.0, 180.0])
    fr = ReferenceFrame(rops, rb, g.positions, g.normals, side, L, 0.25, 8, cam, workers=workers)
    try:
        faces = env.faces(13.0)
        mat = (np.array([1.2, 1.5, 1.8]), np.array([0.01, 0.02, 0.04]), 1.3)
        rad, unc, t, spectra = fr.relight(faces, mat)
        E = O.env_irradiance(O.env_transfer_w2(g.normals.astype(np.float64), 8),
                             O.project_environment(faces, 128))
        ref = O.relight(E, ops, b.bases, b.r_nodes, mat, side, L, "haar", 0.25,
                        g.normals.astype(np.float64), g.positions.astype(np.float64), cam)
        for c in range(3):
            assert np.array_equal(spectra[c].indices, ref["spectra"][c].indices)
        assert np.abs(unc - ref["radiance_unclamped"]).max() <= 1e-12 * np.abs(unc).max()
        assert set(t) == {"irradiance", "transfer", "weighting", "inverse_wavelet"}
        m2 = (np.array([2.0, 2.2, 2.5]), np.array([0.003, 0.01, 0.02]), 1.3)
        rad2, unc2, _ = fr.set_material(m2)
        ref2 = O.relight(E, ops, b.bases, b.r_nodes, m2, side, L, "haar", 0.25,
                         g.normals.astype(np.float64), g.positions.astype(np.float64), cam)
        assert np.abs(unc2 - ref2["radiance_unclamped"]).max() <= 1e-12 * np.abs(unc2).max()
    finally:
        fr.close()
