"""Property tests of the GPU path, mirroring the reference's own test
strategy: wavelet invariants (test_wavelets.py:14-60),
the lossless / monotone / bookkeeping properties of the two-step compression
(test_transfer.py:122-181), and the frame's light linearity and zero light
(test_runtime.py:28-50) — here on the device kernels.
"""

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


# ---- wavelets (test_wavelets.py:14-60) ----------------------------------------
@pytest.mark.parametrize("side,L", [(2, 1), (64, 6), (128, 3), (256, 3)])
def test_haar_roundtrip_parseval_linearity(lib, side, L):
    from paper_2203_12339_b200.wavelets import haar2d, haar2d_inverse

    rng = np.random.default_rng(side + L)
    a = torch.as_tensor(rng.standard_normal((side, side)), device="cuda")
    b = torch.as_tensor(rng.standard_normal((side, side)), device="cuda")
    fa = haar2d(a, L)
    assert torch.allclose(haar2d_inverse(fa, L), a, rtol=0, atol=1e-12)
    assert float((fa * fa).sum()) == pytest.approx(float((a * a).sum()), rel=1e-12)
    lin = haar2d(2.0 * a - 3.0 * b, L)
    assert torch.allclose(lin, 2.0 * fa - 3.0 * haar2d(b, L), rtol=0, atol=1e-11)


def test_haar_constant_is_pure_dc(lib):
    """test_wavelets.py:14-17 / 48-51: a constant grid keeps only the
    coarse band (value * 2^L per coefficient of the LL block), details 0."""
    from paper_2203_12339_b200.wavelets import haar2d

    for side, L in ((2, 1), (32, 5), (64, 3)):
        f = haar2d(torch.full((side, side), 3.0, dtype=torch.float64, device="cuda"), L).cpu().numpy()
        h = side >> L
        assert np.allclose(f[:h, :h], 3.0 * (1 << L), rtol=1e-14)
        f[:h, :h] = 0.0
        assert np.abs(f).max() <= 1e-12


# ---- two-step compression (test_transfer.py:122-181) ----------------------------
def _geo_basis(side=16, K=4):
    from paper_2203_12339_b200.basis import build_basis
    from paper_2203_12339_b200.geometry import make_geometry_image

    return make_geometry_image(side, 10.0, 0.05, 8, 2203), build_basis(K, (4, 4))


def _frame_scatter(g, b, dt, Lsh, e_keep):
    from paper_2203_12339_b200 import config as C
    from paper_2203_12339_b200.basis import OpticalMaterial
    from paper_2203_12339_b200.runtime import Scene, SHLight

    m = OpticalMaterial(sigma_s_prime=C.C1.material[0], sigma_a=C.C1.material[1], eta=1.3)
    sc = Scene(g, dt, b, m, SHLight(Lsh), e_keep=e_keep, keep_scatter=True)
    sc.relight()
    return sc.scatter.cpu().numpy(), m


def _truncated_kernel_scatter(g, b, Lsh, m):
    """The K-truncated kernel oracle (tests/conftest.py:53-61 pattern): dense
    transfer_block rows, no wavelet compression, applied to E, weighted by
    project_material."""
    from paper_2203_12339_b200 import lighting as LT

    pos = g.positions.astype(np.float64)
    area = g.area.astype(np.float64)
    slopes = O.basis_slopes(b.bases, b.r_nodes)
    blk = O.transfer_block(pos, pos, area, b.r_nodes, b.bases, slopes)  # (N, K, N)
    E = O.sh_irradiance(LT.sh_transfer(g.normals, 3), Lsh)               # (N, 3)
    w = O.project_material(b.bases, b.r_nodes, m.sigma_s_prime, m.sigma_a, m.eta)  # (3, K)
    vk = np.einsum("oki,ic->koc", blk, E)
    return np.einsum("ck,koc->oc", w, vk)


def test_lossless_settings_match_truncated_kernel(lib):
    """step1_keep = 1, step2_fraction = 1, e_keep = 1: the compressed frame
    equals the dense truncated-kernel product (the reference bounds it by
    1e-6, test_transfer.py:122-132; f32 operator storage here)."""
    from paper_2203_12339_b200 import lighting as LT
    from paper_2203_12339_b200.precompute import precompute_compressed

    g, b = _geo_basis()
    dt = precompute_compressed(g, b, 2, 1.0, 1.0)
    Lsh = LT.random_sh_light(3, 4)
    got, m = _frame_scatter(g, b, dt, Lsh, 1.0)
    ref = _truncated_kernel_scatter(g, b, Lsh, m)
    assert np.abs(got - ref).max() <= 1e-6 * np.abs(ref).max()


def test_error_monotone_in_fraction_and_energy_bookkeeping(lib):
    """test_transfer.py:162-181: the frame's relative L2 error against the
    lossless frame does not grow as step2_fraction rises; per term kept <=
    total energy, kept >= fraction * total, and the stored values' energy is
    the kept energy (f32 storage: rel 1e-6)."""
    from paper_2203_12339_b200 import lighting as LT
    from paper_2203_12339_b200.precompute import precompute_compressed

    g, b = _geo_basis()
    Lsh = LT.random_sh_light(3, 6)
    ref, m = _frame_scatter(g, b, precompute_compressed(g, b, 2, 1.0, 1.0), Lsh, 1.0)
    errs = []
    for frac in (0.9, 0.99, 0.9999):
        dt = precompute_compressed(g, b, 2, 1.0, frac)
        for k, op in enumerate(dt.to_reference()):
            assert dt.kept_energy[k] <= dt.total_energy[k] * (1 + 1e-12)
            assert dt.kept_energy[k] >= frac * dt.total_energy[k] * (1 - 1e-12)
            assert float(np.sum(op.vals ** 2)) == pytest.approx(dt.kept_energy[k], rel=1e-6)
        got, _ = _frame_scatter(g, b, dt, Lsh, 1.0)
        errs.append(np.linalg.norm(got - ref) / np.linalg.norm(ref))
    assert errs[0] >= errs[1] >= errs[2], errs


# ---- frame (test_runtime.py:28-50) --------------------------------------------------
def test_zero_light_zero_frame_and_doubling(lib):
    from paper_2203_12339_b200 import lighting as LT
    from paper_2203_12339_b200.precompute import precompute_compressed

    g, b = _geo_basis(32)
    dt = precompute_compressed(g, b, 2, 0.10, 0.95)
    Lsh = LT.random_sh_light(3, 2)
    s0, _ = _frame_scatter(g, b, dt, np.zeros_like(Lsh), 0.25)
    assert np.all(s0 == 0.0)
    s1, _ = _frame_scatter(g, b, dt, Lsh, 0.25)
    s2, _ = _frame_scatter(g, b, dt, 2.0 * Lsh, 0.25)
    assert np.abs(s2 - 2.0 * s1).max() <= 1e-12 * np.abs(s1).max()
