"""Parity at BASELINE's own sizes: the medium interactive
config C2 (128^2, K=8, SH order 5, per-frame SO(3) rotation + new material)
end to end against the oracle on the GPU-built operator, and the
environment-lit large mesh C3 (256^2, the bench workload) through the
size-independent properties: sampled receiver rows of v_k against the
oracle's CSR apply of the same operator and spectrum, stages 3-5 on the full
v_k against the oracle's finish, kept sets identical to the oracle's top-n of
the device E, linearity in the light, edit == relight.

Bars as the rest of the suite: kept index sets identical; radiance within
1e-4 under the tau = 1e-3 floor.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import sss_oracle as O  # noqa: E402

TOL = 1e-4
TAU = 1e-3


@pytest.fixture(scope="module")
def lib():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    from paper_2203_12339_b200 import _lib, build

    build.build()
    return _lib.load()


def _setup(cfg):
    from paper_2203_12339_b200.basis import build_basis
    from paper_2203_12339_b200.geometry import from_config
    from paper_2203_12339_b200.precompute import precompute_compressed

    g = from_config(cfg)
    b = build_basis(cfg.K, cfg.lattice)
    dt = precompute_compressed(g, b, cfg.levels, cfg.step1_keep, cfg.step2_fraction)
    return g, b, dt


def _material(rng, eta=1.3):
    from paper_2203_12339_b200.basis import OpticalMaterial

    lu = lambda lo, hi: np.exp(rng.uniform(np.log(lo), np.log(hi), 3))  # noqa: E731
    return OpticalMaterial(sigma_s_prime=lu(0.5, 3.0), sigma_a=lu(0.001, 0.05), eta=eta)


def test_c2_frames_parity(lib):
    """BASELINE configs[1]: frames with a seeded uniform SO(3) rotation of the
    SH light and a new log-uniform material each, against the oracle frame
    on the same (GPU-precomputed, f32-stored) operator."""
    from paper_2203_12339_b200 import config as C
    from paper_2203_12339_b200 import lighting as LT
    from paper_2203_12339_b200.runtime import Scene, SHLight

    cfg = C.C2
    g, b, dt = _setup(cfg)
    ops = dt.to_reference()
    L0 = LT.random_sh_light(cfg.sh_bands, 11)
    rng = np.random.default_rng(12)
    sc = Scene(g, dt, b, _material(rng), SHLight(L0), keep_scatter=True)
    T = LT.sh_transfer(g.normals, cfg.sh_bands)
    for f in range(3):
        L = LT.rotate_sh(L0, LT.random_rotation(rng))
        m = _material(rng)
        sc.set_light(SHLight(L))
        fr = sc.set_material(m)
        E = O.sh_irradiance(T, L)
        ref = O.relight(E, ops, b.bases, b.r_nodes, (m.sigma_s_prime, m.sigma_a, m.eta),
                        cfg.side, cfg.levels, "haar", C.E_KEEP, g.normals.astype(np.float64),
                        g.positions.astype(np.float64), np.array(C.CAMERA[0]))
        for c in range(3):
            assert np.array_equal(sc.selected_indices(c), ref["spectra"][c].indices), (f, c)
        assert O.parity_error(fr.radiance_unclamped, ref["radiance_unclamped"], TAU) <= TOL, f
        assert O.parity_error(sc.scatter.cpu().numpy(), ref["scatter"], TAU) <= TOL, f


@pytest.fixture(scope="module")
def c3(lib):
    from paper_2203_12339_b200 import config as C
    from paper_2203_12339_b200 import lighting as LT
    from paper_2203_12339_b200.runtime import EnvLight, Scene

    cfg = C.C3
    g, b, dt = _setup(cfg)
    env = LT.Environment(side=cfg.env_side, seed=7)
    rng = np.random.default_rng(5)
    sc = Scene(g, dt, b, _material(rng), EnvLight(env.faces(0.0)), e_keep=cfg.e_keep,
               keep_scatter=True)
    return cfg, g, b, dt, env, sc


def test_c3_transfer_rows_and_finish_vs_oracle(c3):
    """Full-size C3 frame: the device E's top-n sets equal the oracle's
    selection of the same E; v_k on 512 sampled receiver rows equals the
    oracle's CSR apply of the same operator to the device's kept spectrum;
    stages 3-5 on the full device v_k equal the oracle's finish."""
    from paper_2203_12339_b200 import config as C
    from paper_2203_12339_b200.runtime import EnvLight
    from paper_2203_12339_b200.transfer import tile_major_to_flat

    cfg, g, b, dt, env, sc = c3
    sc.set_light(EnvLight(env.faces(17.0)))
    fr = sc.relight()
    sc._launch_stage1(want_E=True)  # the same stage 1 again, keeping E (N, 3)
    torch.cuda.synchronize()
    E = sc.E.cpu().numpy()
    n = dt.n
    perm = tile_major_to_flat(cfg.side, cfg.levels)       # tile-major -> flat
    x = sc.x.cpu().numpy()                                  # (3, N) tile-major kept spectrum
    vk = sc.vk.cpu().numpy()                                # (K, 3, N) tile-major
    rng = np.random.default_rng(9)
    rows = np.sort(rng.choice(n, 512, replace=False))
    rp = dt.rowptr.cpu().numpy()
    cols = dt.cols.cpu().numpy().view(np.uint32)
    vals = dt.vals.cpu().numpy()
    for k in range(dt.K):
        ref = O.csr_rows_apply(rp[k], cols, vals, rows, x)  # (rows, 3)
        got = vk[k][:, rows].T
        scale = np.abs(vk[k]).max()
        assert np.abs(got - ref).max() <= 1e-12 * scale, k
    # stages 3-5 on the full v_k (flat order for the oracle)
    vk_flat = vk[:, :, np.argsort(perm)]
    m = sc.material
    w = O.project_material(b.bases, b.r_nodes, m.sigma_s_prime, m.sigma_a, m.eta)
    rad, unc, scatter = O.finish(vk_flat, w, cfg.side, cfg.levels, "haar",
                                 g.normals.astype(np.float64), g.positions.astype(np.float64),
                                 np.array(C.CAMERA[0]), m.eta)
    assert O.parity_error(fr.radiance_unclamped, unc, TAU) <= TOL
    assert O.parity_error(sc.scatter.cpu().numpy(), scatter, TAU) <= TOL
    # the kept sets: the oracle's top-n of the device's own E
    spectra = O.select_irradiance(E, cfg.side, cfg.levels, cfg.e_keep)
    for c in range(3):
        assert np.array_equal(sc.selected_indices(c), spectra[c].indices)
    keep = max(1, int(round(cfg.e_keep * n)))
    for c in range(3):
        assert sc.selected_indices(c).size == keep


def test_c3_linearity_and_edit_equals_relight(c3):
    """Doubling the environment doubles the frame (the top-n sets are scale
    invariant, the path is linear in the light); a material edit through the
    cached v_k equals a full relight with that material."""
    from paper_2203_12339_b200.runtime import EnvLight

    cfg, g, b, dt, env, sc = c3
    faces = env.faces(42.0)
    a = sc.set_light(EnvLight(faces))
    d = sc.set_light(EnvLight(2.0 * faces))
    assert np.abs(d.radiance_unclamped - 2.0 * a.radiance_unclamped).max() <= \
        1e-6 * np.abs(a.radiance_unclamped).max()
    m = _material(np.random.default_rng(77))
    edited = sc.set_material(m)
    full = sc.relight()
    assert np.abs(edited.radiance - full.radiance).max() <= 1e-6 * np.abs(full.radiance).max()
