"""The kernel seam on the GPU (`_accel.get_kernels()`,
_accel.py:35-43): ``paper_2203_12339_b200.kernels_b200`` has the signatures
of the reference's ``_kernels_nb`` and must reproduce it BITWISE.

* each kernel against the oracle's restatement (pinned to the reference by
  tests/test_oracle_golden.py) on seeded inputs, at the reference test sizes
  and at geometry-image sizes (256^2 grids, 9/7 full pyramid);
* the reference's own test suite (baseline/_ref/ref_pkg/tests, installed by
  tools/install_reference.sh) run with the GPU module swapped in behind the
  seam (tests/reference_seam_plugin.py): test_kernels.py then compares the
  GPU kernels with the reference's numpy twins, and test_wavelets /
  test_transfer / test_runtime / test_lighting / test_container drive them
  through the reference's own callers (precompute, Scene.relight, shadows).
"""

import json
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import sss_oracle as O  # noqa: E402

ROOT = Path(__file__).resolve().parents[1]
REF = ROOT / "baseline" / "_ref"
REF_PKG = REF / "ref_pkg"


@pytest.fixture(scope="module")
def kb():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    from paper_2203_12339_b200 import build

    build.build()
    from paper_2203_12339_b200 import kernels_b200

    return kernels_b200


@pytest.mark.gpu
@pytest.mark.parametrize("shape", [(4, 32, 32), (3, 2, 2), (1, 1, 1), (2, 256, 256), (5, 64, 64)])
def test_wavelets_bitwise(kb, shape):
    rng = np.random.default_rng(sum(shape))
    x = rng.standard_normal(shape)
    assert np.array_equal(kb.haar2d_fwd_batch(x), O.haar2d_fwd(x))
    assert np.array_equal(kb.haar2d_inv_batch(x), O.haar2d_inv(x))
    assert np.array_equal(kb.cdf97_fwd_batch(x), O.cdf97_fwd(x))
    assert np.array_equal(kb.cdf97_inv_batch(x), O.cdf97_inv(x))


@pytest.mark.gpu
def test_wavelet_round_trip_and_float32_input(kb):
    rng = np.random.default_rng(3)
    x = rng.standard_normal((8, 128, 128)).astype(np.float32)
    assert np.array_equal(kb.cdf97_fwd_batch(x), O.cdf97_fwd(x.astype(np.float64)))
    y = kb.cdf97_inv_batch(kb.cdf97_fwd_batch(x))
    assert np.abs(y - x).max() < 1e-5
    h = kb.haar2d_inv_batch(kb.haar2d_fwd_batch(x))
    assert np.abs(h - x).max() < 1e-5


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_transfer_block_bitwise(kb, dtype):
    rng = np.random.default_rng(11)
    n, k, nr = 700, 6, 64
    positions = (rng.random((n, 3)) * 40.0).astype(dtype)
    areas = rng.random(n) + 0.1
    r_nodes = np.concatenate([[0.0], np.sort(rng.random(nr - 1)) * 60.0])
    bases = rng.standard_normal((k, nr))
    slopes = (bases[:, 1:] - bases[:, :-1]) / np.diff(r_nodes)
    block = positions[100:164]
    got = kb.transfer_block(block, positions, areas, r_nodes, bases, slopes)
    want = O.transfer_block(block, positions, areas, r_nodes, bases, slopes)
    assert got.shape == (64, k, n) and got.dtype == np.float64
    assert np.array_equal(got, want)


@pytest.mark.gpu
def test_csc_apply_bitwise(kb):
    rng = np.random.default_rng(5)
    for n_cols, out_len, nx in [(50, 512, 100), (3000, 20000, 4000), (1, 7, 1)]:
        cols = np.sort(rng.choice(4 * n_cols + 8, n_cols, replace=False)).astype(np.uint32)
        counts = rng.integers(0, 40, n_cols)
        colptr = np.zeros(n_cols + 1, np.int64)
        colptr[1:] = np.cumsum(counts)
        nnz = int(colptr[-1])
        rowidx = rng.integers(0, out_len, nnz).astype(np.uint32)  # repeats within a column
        vals = rng.standard_normal(nnz)
        x_idx = np.sort(rng.choice(4 * n_cols + 8, min(nx, 4 * n_cols + 8),
                                   replace=False)).astype(np.uint32)
        x_val = rng.standard_normal(x_idx.size)
        want = O.csc_apply(cols, colptr, rowidx, vals, x_idx, x_val, out_len)
        for _ in range(2):  # the second call hits the cached device operator
            got = kb.csc_apply(cols, colptr, rowidx, vals, x_idx, x_val, out_len)
            assert np.array_equal(got, want)
    # no active column / empty spectrum / float32 values
    cols = np.array([5, 9], np.uint32)
    colptr = np.array([0, 2, 3], np.int64)
    rowidx = np.array([1, 2, 3], np.uint32)
    vals = np.array([1.0, 2.0, 3.0], np.float32)
    assert kb.csc_apply(cols, colptr, rowidx, vals, np.array([7], np.uint32), np.array([4.0]), 8).sum() == 0.0
    assert kb.csc_apply(cols, colptr, rowidx, vals, np.zeros(0, np.uint32), np.zeros(0), 8).sum() == 0.0
    got = kb.csc_apply(cols, colptr, rowidx, vals, np.array([9], np.uint32), np.array([0.1]), 8)
    assert np.array_equal(got, O.csc_apply(cols, colptr, rowidx, vals.astype(np.float64),
                                           np.array([9], np.uint32), np.array([0.1]), 8))
    with pytest.raises(ValueError):
        kb.csc_apply(cols, colptr, rowidx, vals, np.array([9, 5], np.uint32), np.ones(2), 8)


@pytest.mark.gpu
def test_raster_fill_bitwise(kb):
    rng = np.random.default_rng(9)
    n_tris = 300
    nv = 3 * n_tris
    tris = np.arange(nv, dtype=np.int64).reshape(n_tris, 3)
    tris[50:60] = tris[40:50]  # duplicate triangles: depth ties
    sx = rng.uniform(-10, 138, nv)
    sy = rng.uniform(-10, 106, nv)
    zn = rng.uniform(0.5, 5.0, nv)
    iw = rng.uniform(0.2, 2.0, nv)
    iw[rng.random(nv) < 0.1] = 0.0
    colors = rng.random((nv, 3))
    img_a, zb_a = np.zeros((96, 128, 3)), np.full((96, 128), np.inf)
    zb_a[:20, :30] = 1.0
    img_b, zb_b = img_a.copy(), zb_a.copy()
    O.raster_fill(tris, sx, sy, zn, iw, colors, zb_a, img_a)
    ret = kb.raster_fill(tris, sx, sy, zn, iw, colors, zb_b, img_b)
    assert ret is zb_b
    assert np.array_equal(img_a, img_b)
    assert np.array_equal(zb_a, zb_b)


@pytest.mark.gpu
def test_bvh_any_hit_matches_reference(kb):
    if not (REF / "sssrelight").exists():
        pytest.skip("baseline/_ref not installed (tools/install_reference.sh)")
    sys.path.insert(0, str(REF))
    try:
        from sssrelight import _kernels_np as knp
        from sssrelight.lighting import build_accelerator
        from sssrelight.meshgen import make_torus
    finally:
        sys.path.remove(str(REF))
    accel = build_accelerator(make_torus())
    rng = np.random.default_rng(21)
    n = 20000
    origins = rng.uniform(-50, 50, (n, 3))
    dirs = rng.standard_normal((n, 3))
    dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
    tmax = rng.uniform(1.0, 200.0, n)
    args = (origins, dirs, tmax, accel.node_min, accel.node_max, accel.node_left,
            accel.node_right, accel.node_start, accel.node_count, accel.v0, accel.e1, accel.e2)
    got = kb.bvh_any_hit(*args)
    assert got.dtype == np.bool_ and got.any() and not got.all()
    assert np.array_equal(got, knp.bvh_any_hit(*args))


def _run_reference_suite(module: str, files, tmp_path):
    if not (REF_PKG / "tests").exists():
        pytest.skip("reference tests not installed (tools/install_reference.sh)")
    counts = tmp_path / "counts.json"
    env = dict(os.environ, SSS_SEAM_MODULE=module, SSS_SEAM_COUNTS=str(counts),
               PYTHONPATH=os.pathsep.join([str(REF), str(ROOT), str(ROOT / "tests")]))
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "reference_seam_plugin",
                        "-p", "no:cacheprovider", *files], cwd=REF_PKG, env=env,
                       capture_output=True, text=True, timeout=1500)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    return json.loads(counts.read_text()), r.stdout


def test_seam_swap_routes_reference_calls(tmp_path):
    """CPU check of the swap mechanism: a call-counting wrapper of the
    reference's numpy kernels is swapped in; the reference's callers must
    route every hot loop through it."""
    counts, _ = _run_reference_suite("sssrelight._kernels_np",
                                     ["tests/test_kernels.py", "tests/test_wavelets.py"], tmp_path)
    for name in ("haar2d_fwd_batch", "cdf97_fwd_batch", "csc_apply", "transfer_block",
                 "bvh_any_hit", "raster_fill"):
        assert counts.get(name, 0) > 0, (name, counts)


@pytest.mark.gpu
def test_reference_suite_through_gpu_seam(kb, tmp_path):
    """The reference's own tests, their callers bound to the GPU kernels."""
    files = ["tests/test_kernels.py", "tests/test_wavelets.py", "tests/test_transfer.py",
             "tests/test_runtime.py", "tests/test_lighting.py", "tests/test_container.py"]
    counts, out = _run_reference_suite("paper_2203_12339_b200.kernels_b200", files, tmp_path)
    for name in ("haar2d_fwd_batch", "haar2d_inv_batch", "cdf97_fwd_batch", "cdf97_inv_batch",
                 "transfer_block", "bvh_any_hit", "csc_apply", "raster_fill"):
        assert counts.get(name, 0) > 0, (name, counts)
    assert " passed" in out
