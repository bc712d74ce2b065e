"""Pin the CPU oracle to the real reference: every check below compares
``oracle/sss_oracle.py`` with fixtures produced by running the reference itself
(tests/golden/make_golden.py). CPU only."""

import numpy as np
import pytest

from oracle import sss_oracle as O
from pathlib import Path

GOLDEN = Path(__file__).resolve().parent / "golden"


def test_haar_full_pyramid_bitwise(golden):
    g = golden("wavelets")
    assert np.array_equal(O.haar2d_fwd(g["x"]), g["haar_fwd"])
    assert np.array_equal(O.haar2d_inv(g["x"]), g["haar_inv"])


@pytest.mark.parametrize("L", [1, 2, 3])
def test_haar_level_limited_bitwise(golden, L):
    g = golden("wavelets")
    assert np.array_equal(O.haar2d_fwd(g["x"], L), g[f"haar_fwd_L{L}"])
    assert np.array_equal(O.haar2d_inv(g["x"], L), g[f"haar_inv_L{L}"])


def test_haar_full_levels_equals_default(golden):
    g = golden("wavelets")
    assert np.array_equal(O.haar2d_fwd(g["x"], 5), g["haar_fwd"])


def test_cdf97_bitwise(golden):
    g = golden("wavelets")
    assert np.array_equal(O.cdf97_fwd(g["x"]), g["cdf_fwd"])
    assert np.array_equal(O.cdf97_inv(g["x"]), g["cdf_inv"])


def test_level_limited_roundtrip():
    x = np.random.default_rng(0).standard_normal((3, 64, 64))
    for L in range(0, 7):
        y = O.haar2d_inv(O.haar2d_fwd(x, L), L)
        assert np.abs(y - x).max() < 1e-12


def test_level_limited_is_tile_local():
    """L-level Haar of a 2^L x 2^L tile depends only on that tile (the
    property the fused inverse-Haar epilogue relies on)."""
    rng = np.random.default_rng(1)
    x = rng.standard_normal((1, 32, 32))
    y = x.copy()
    y[0, 8:16, 16:24] += rng.standard_normal((8, 8))
    d = O.haar2d_fwd(y, 3) - O.haar2d_fwd(x, 3)
    changed = np.argwhere(np.abs(d[0]) > 0)
    # every changed coefficient belongs to spatial tile (1, 2)
    for r, c in changed:
        assert O.coeff_tile(r, c, 32, 3) == (1, 2)
    assert len(changed) == 64


def test_selection_bitwise(golden):
    g = golden("select")
    v = g["v"]
    for n in (0, 1, 7, 410, 1024, 4096):
        s = O.compress_top_n(v, n)
        assert np.array_equal(s.indices, g[f"top_{n}_idx"])
        assert np.array_equal(s.values, g[f"top_{n}_val"])
        assert np.array_equal([s.total_energy, s.kept_energy], g[f"top_{n}_e"])
    for f in (0.0, 0.5, 0.9, 0.95, 0.9999, 1.0):
        s = O.compress_energy(v, f)
        assert np.array_equal(s.indices, g[f"en_{f}_idx"])
        assert np.array_equal([s.total_energy, s.kept_energy], g[f"en_{f}_e"])


def test_selection_worked_examples():
    # wavelets tests: tests/test_wavelets.py:153-179
    assert list(O.compress_top_n(np.array([3.0, -5.0, 2.0]), 1).indices) == [1]
    assert list(O.compress_top_n(np.array([2.0, -2.0, 2.0]), 2).indices) == [0, 1]
    s = O.compress_energy(np.array([3.0, 2.0, 1.0]), 0.9)
    assert list(s.indices) == [0, 1] and s.kept_energy == 13.0
    assert O.compress_energy(np.array([3.0, 0.0, 2.0, 1.0]), 1.0).count == 3


def test_dipole_bitwise(golden):
    g = golden("dipole")
    rd = [float(O.eval_rd(O.derive_dipole_raw(a, b, c), r)) for a, b, c, r in g["pts"]]
    assert np.array_equal(rd, g["rd"])
    for i, e in enumerate((1.0, 1.2, 1.3, 1.5)):
        assert np.array_equal(O.fresnel_transmittance(e, g["cos"]), g["ft"][i])
        assert O.fdr(e) == g["fdr"][i]


@pytest.mark.parametrize("key,lat,K", [("4x4_K4", (4, 4), 4), ("8x4_K8", (8, 4), 8),
                                       ("8x8_K12", (8, 8), 12), ("8x8_K8", (8, 8), 8)])
def test_basis_matches_reference(golden, key, lat, K):
    from paper_2203_12339_b200 import config as C

    g = golden("basis")
    r_nodes = O.r_nodes_for_box(C.SIGMA_BOX, C.ETA)
    assert np.array_equal(r_nodes, g["r_nodes"])
    nodes = O.sigma_lattice(C.SIGMA_BOX, *lat)
    bases, sv, U = O.decompose(O.assemble_matrix(r_nodes, nodes, C.ETA), r_nodes, K)
    # same LAPACK here; SVD values are parity-unpinned across builds
    scale = np.abs(g[f"{key}_bases"]).max()
    assert np.abs(bases - g[f"{key}_bases"]).max() <= 1e-9 * scale
    assert np.allclose(sv, g[f"{key}_sv"], rtol=1e-10)
    s = O.project_material(bases, r_nodes, *C.C1.material)
    assert np.allclose(s, g[f"{key}_s"], rtol=1e-8, atol=1e-12)


def test_exact_projection_reproduces_nodes(golden):
    """b_k(r_j) == sum_m P[k,m] R_d(r_j; sigma_m) (SURVEY §8c exact mode)."""
    from paper_2203_12339_b200 import config as C

    g = golden("basis")
    r_nodes = g["r_nodes"]
    nodes = O.sigma_lattice(C.SIGMA_BOX, 8, 8)
    bases, sv, U = O.decompose(O.assemble_matrix(r_nodes, nodes, C.ETA), r_nodes, 8)
    P = O.exact_projection_coeffs(U, sv, r_nodes, 8)
    rd = np.stack([O.eval_rd(O.derive_dipole_raw(a, b, C.ETA), r_nodes) for a, b in nodes])
    assert np.abs(P @ rd - bases).max() <= 1e-8 * np.abs(bases).max()


def test_transfer_block_and_csc_bitwise(golden):
    g = golden("kernels")
    bases = g["bases"]
    slopes = O.basis_slopes(bases, g["r_nodes"])
    rows = O.transfer_block(g["positions"][:8], g["positions"], g["areas"], g["r_nodes"],
                            bases, slopes)
    assert np.array_equal(rows, g["rows"])
    out = O.csc_apply(g["cols"], g["colptr"], g["rowidx"], g["vals"], g["x_idx"],
                      g["x_val"], 512)
    assert np.array_equal(out, g["csc_out"])


def _gi16():
    from paper_2203_12339_b200.geometry import make_geometry_image

    gi = make_geometry_image(16, amp=0.05, seed=11)
    return (gi.positions.astype(np.float64), gi.normals.astype(np.float64),
            gi.area.astype(np.float64))


@pytest.mark.parametrize("frac", [0.95, 0.9999])
def test_precompute_full_pyramid_cdf97_bitwise(golden, frac):
    """The restated two-step compression at (levels=full, w1=9/7) IS the
    reference's precompute_compressed (transfer.py:350-361), bit for bit."""
    g = golden("precompute16")
    b = golden("basis")
    pos, _, area = _gi16()
    ops = O.precompute_compressed(pos, area, 16, b["r_nodes"], b["4x4_K4_bases"], 0.1, frac,
                                  levels=None, w1="cdf97")
    for ki, op in enumerate(ops):
        tag = f"k0.1_f{frac}_op{ki}"
        assert np.array_equal(op.cols, g[f"{tag}_cols"])
        assert np.array_equal(op.colptr, g[f"{tag}_colptr"])
        assert np.array_equal(op.rowidx, g[f"{tag}_rowidx"])
        assert np.array_equal(op.vals, g[f"{tag}_vals"])
        assert np.array_equal([op.kept_energy, op.total_energy, op.step1_entries],
                              g[f"{tag}_e"])


def test_frame_full_pyramid_cdf97_bitwise(golden):
    g = golden("precompute16")
    b = golden("basis")
    pos, nrm, area = _gi16()
    ops = O.precompute_compressed(pos, area, 16, b["r_nodes"], b["4x4_K4_bases"], 0.1, 0.95,
                                  levels=None, w1="cdf97")
    from paper_2203_12339_b200 import config as C

    out = O.relight(g["E"], ops, b["4x4_K4_bases"], b["r_nodes"], C.C1.material, 16, None,
                    "cdf97", 0.25, nrm, pos, np.array([0.0, 0.0, 180.0]))
    for c in range(3):
        assert np.array_equal(out["spectra"][c].indices, g[f"E_idx{c}"])
    assert np.allclose(out["vk"], g["vk"], rtol=0, atol=1e-15 * np.abs(g["vk"]).max())
    assert np.allclose(out["radiance_unclamped"], g["unclamped"], rtol=1e-12,
                       atol=1e-14 * np.abs(g["unclamped"]).max())


def test_env_projection_matches_reference(golden):
    g = golden("env")
    spectra = O.project_environment(g["faces"], 32)
    for c in range(3):
        assert np.array_equal(spectra[c].indices, g[f"idx{c}"])
        assert np.array_equal(spectra[c].values, g[f"val{c}"])
    _, nrm, _ = _gi16()
    W = O.visibility_weights(nrm, 8)
    assert np.allclose(W, g["W"], rtol=1e-14, atol=1e-18)
    w2 = O.haar2d_fwd(W.reshape(-1, 8, 8)).reshape(W.shape[0], -1)
    E = O.env_irradiance(w2, spectra)  # fp64 w2 here: Parseval identity
    assert np.allclose(E, g["E"], rtol=1e-11, atol=1e-14)


def test_direct_lights_oracle_matches_reference(golden):
    """irradiance_direct (point + directional + sphere light, BVH shadow rays)
    and any-hit queries, against the reference run on the geometry image's
    grid mesh (lighting.py:101-290)."""
    g = golden("direct")
    h = O.any_hit(g["ray_o"], g["ray_d"], g["ray_t"], g["positions"], g["triangles"])
    assert np.array_equal(h, g["hits"])
    lights = [("point", g["p_pos"], g["p_int"]), ("directional", g["d_dir"], g["d_irr"]),
              ("sphere", g["s_c"], float(g["s_r"]), g["s_rad"])]
    E = O.irradiance_direct(g["positions"], g["normals"], lights, g["positions"], g["triangles"],
                            float(g["eta"]))
    assert np.array_equal(E, g["E"])


def test_fold_oracle_matches_reference(golden):
    """precompute_visibility + fold_visibility + the folded ambient apply
    (transfer.py:368-451, runtime.py:146-149) against the reference's own
    output on a self-occluding 16^2 geometry (96 directions): visibility,
    folded operators (sets, values, energy ledgers) and v_k bitwise."""
    g = golden("fold")
    d = golden("direct")
    vis = O.precompute_visibility(d["positions"], d["normals"], d["positions"], d["triangles"],
                                  int(g["face_side"]))
    assert np.array_equal(vis.astype(np.uint8), g["vis"])
    assert 0.2 < vis.mean() < 0.8  # genuinely self-occluding
    K = 4
    ops = [O.Operator(g[f"op{k}_cols"], g[f"op{k}_colptr"], g[f"op{k}_rowidx"], g[f"op{k}_vals"],
                      float(g[f"op{k}_e"][0]), float(g[f"op{k}_e"][1]), int(g[f"op{k}_e"][2]))
           for k in range(K)]
    folded, _ = O.fold_visibility(ops, g["vis"].astype(np.float64), d["normals"], int(g["side"]),
                                  int(g["face_side"]), float(g["eta"]), float(g["fraction"]))
    for k, f in enumerate(folded):
        for name in ("cols", "colptr", "rowidx", "vals"):
            assert np.array_equal(getattr(f, name), g[f"fold{k}_{name}"]), (k, name)
        assert [f.kept_energy, f.total_energy, f.step1_entries] == g[f"fold{k}_e"].tolist()
    spec = [O.Spectrum(g[f"env_idx{c}"], g[f"env_val{c}"], 96, 0.0, 0.0) for c in range(3)]
    assert np.array_equal(O.ambient_vk(folded, spec, int(g["side"]) ** 2), g["vk"])
    # zero visibility folds to zero operators (test_transfer.py:265-273)
    zero, _ = O.fold_visibility(ops, np.zeros_like(vis), d["normals"], int(g["side"]),
                                int(g["face_side"]), 1.3)
    assert all(z.cols.size == 0 and z.rowidx.size == 0 for z in zero)


def test_raster_oracle_matches_reference(golden):
    """raster_fill / _project_vertices / render_image quantisation
    (runtime.py:230-273, _kernels_np.py:264-313) against the reference run on
    the same inputs: images and z-buffers bitwise; the projection (BLAS
    matmul in the reference, ordered sums here) to 1e-12 and, fed the
    reference's own projected vertices, the raster is bitwise."""
    g = golden("raster")
    zb, img = g["r_zbuf0"].copy(), g["r_img0"].copy()
    O.raster_fill(g["r_tris"], g["r_sx"], g["r_sy"], g["r_zn"], g["r_iw"], g["r_colors"], zb, img)
    assert np.array_equal(zb, g["r_zbuf"]) and np.array_equal(img, g["r_img"])
    for ci in range(2):
        pos, at, fov = g[f"c{ci}_pos"], g[f"c{ci}_at"], float(g[f"c{ci}_fov"])
        sx, sy, zn, iw = O.project_vertices(g["m_vertices"], pos, at, [0.0, 1.0, 0.0], fov, 96, 72)
        for a, name in ((sx, "sx"), (sy, "sy"), (zn, "zn"), (iw, "iw")):
            ref = g[f"c{ci}_{name}"]
            assert np.allclose(a, ref, rtol=1e-12, atol=1e-12), name
        zb = np.full((72, 96), np.inf)
        img = np.empty((72, 96, 3))
        img[:] = (0.02, 0.02, 0.03)
        O.raster_fill(g["m_tris"], g[f"c{ci}_sx"], g[f"c{ci}_sy"], g[f"c{ci}_zn"], g[f"c{ci}_iw"],
                      g["m_radiance"], zb, img)
        assert np.array_equal(img, g[f"c{ci}_img"]) and np.array_equal(zb, g[f"c{ci}_zbuf"])
        assert np.array_equal(O.encode_srgb8(img, 2.0), g[f"c{ci}_u8"])
        assert np.isfinite(zb).mean() > 0.2  # the object covers the frame


def test_c2_digest_inputs_are_the_config():
    """tests/golden/c2_inputs.npz holds exactly the C2 geometry image and PCA
    basis this container builds from the frozen config (the GPU digest test
    uses the stored copy so the box's numpy cannot change a bit)."""
    import json

    from paper_2203_12339_b200 import config as C
    from paper_2203_12339_b200.basis import build_basis
    from paper_2203_12339_b200.geometry import make_geometry_image

    z = np.load(GOLDEN / "c2_inputs.npz")
    cfg = C.C2
    g = make_geometry_image(cfg.side, cfg.radius, cfg.bump_amp, cfg.bump_terms, cfg.seed)
    b = build_basis(cfg.K, cfg.lattice)
    assert np.array_equal(z["positions"], g.positions) and np.array_equal(z["area"], g.area)
    assert np.array_equal(z["bases"], b.bases) and np.array_equal(z["r_nodes"], b.r_nodes)
    d = json.loads((GOLDEN / "c2_digests.json").read_text())
    assert d["config"] == cfg.name and d["K"] == cfg.K and d["levels"] == cfg.levels
    assert len(d["operators"]) == cfg.K
