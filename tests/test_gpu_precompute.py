"""GPU parity of the offline pair pass and two-step compression (path d)
against the CPU oracle (itself pinned bit-for-bit to the reference's
precompute_compressed, tests/test_oracle_golden.py)."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import sss_oracle as O  # noqa: E402
from paper_2203_12339_b200 import config as C  # noqa: E402


@pytest.fixture(scope="module")
def lib():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    from paper_2203_12339_b200 import _lib, build

    build.build()
    return _lib.load()


def _setup(cfg, side=None, amp=None):
    from paper_2203_12339_b200.basis import build_basis
    from paper_2203_12339_b200.geometry import make_geometry_image

    side = side or cfg.side
    g = make_geometry_image(side, cfg.radius, cfg.bump_amp if amp is None else amp, 8, cfg.seed)
    b = build_basis(cfg.K, cfg.lattice)
    return g, b


def _rows_tm(points, side, L):
    T = 1 << L
    r, c = points // side, points % side
    tile = (r // T) * (side // T) + c // T
    return tile * T * T + (r % T) * T + (c % T)


@pytest.mark.parametrize("side,L", [(32, 2), (64, 3)])
def test_pair_pass_lerp_bitwise(lib, side, L):
    from paper_2203_12339_b200.precompute import PairPass, _tables

    g, b = _setup(C.C2, side)
    n = side * side
    pp = PairPass(g, b, L, exact=False)
    D = torch.empty((n, n), dtype=torch.float64, device="cuda")
    M = torch.empty((n, n), dtype=torch.float64, device="cuda")
    f2t, t2f = _tables(side, L, "cuda")
    f2t = f2t.cpu().numpy()
    pos, area = g.positions.astype(np.float64), g.area.astype(np.float64)
    slopes = O.basis_slopes(b.bases, b.r_nodes)
    rng = np.random.default_rng(side)
    pts = rng.choice(n, 16, replace=False)
    for k in (0, b.K - 1):
        pp.run(k, D, M)
        Dh = D.cpu().numpy()
        rows = O.transfer_block(pos[pts], pos, area, b.r_nodes, b.bases, slopes)[:, k]
        want = O.haar2d_fwd(rows.reshape(-1, side, side), L).reshape(len(pts), n)
        got = Dh[_rows_tm(pts, side, L)][:, f2t]
        assert np.array_equal(got, want)
        # M columns = w1 Haar over receivers of f32(D) (transfer.py:282-322)
        cols = rng.choice(n, 8, replace=False)
        full = O.transfer_block(pos, pos, area, b.r_nodes, b.bases, slopes)[:, k]
        Dfull = O.haar2d_fwd(full.reshape(-1, side, side), L).reshape(n, n)
        colv = Dfull[:, cols].T.astype(np.float32).astype(np.float64)
        wantM = O.haar2d_fwd(colv.reshape(-1, side, side), L).reshape(len(cols), n)
        Mh = M.cpu().numpy()
        gotM = Mh[f2t[cols]][:, f2t]
        assert np.array_equal(gotM, wantM)


def _assert_operators_equal(dt, ops, stats=None):
    got = dt.to_reference()
    for k, (a, o) in enumerate(zip(got, ops)):
        assert np.array_equal(a.cols, o.cols), k  # the step-1 union (step1_unions)
        assert np.array_equal(a.colptr, o.colptr), k
        assert np.array_equal(a.rowidx, o.rowidx), k  # per-column kept row sets, identical
        assert np.array_equal(a.vals, o.vals.astype(np.float32).astype(np.float64))
        assert dt.nnz_per_k[k] == o.nnz
        assert dt.kept_energy[k] == pytest.approx(o.kept_energy, rel=1e-12)
        assert dt.total_energy[k] == pytest.approx(o.total_energy, rel=1e-12)
        if stats is not None:
            assert stats["union_sizes"][k] == o.cols.size
        assert dt.step1_entries[k] == o.step1_entries


@pytest.mark.parametrize("side,L,keep,K", [(32, 2, 0.10, 4), (64, 3, 0.05, 8)])
def test_precompute_matches_oracle(lib, side, L, keep, K):
    from paper_2203_12339_b200.basis import build_basis
    from paper_2203_12339_b200.geometry import make_geometry_image
    from paper_2203_12339_b200.precompute import precompute_compressed

    g = make_geometry_image(side, 10.0, 0.05, 8, 2203)
    b = build_basis(K, (4, 4) if K == 4 else (8, 4))
    stats = {}
    dt = precompute_compressed(g, b, L, keep, C.STEP2_FRACTION, stats=stats)
    ops = O.precompute_compressed(g.positions.astype(np.float64), g.area.astype(np.float64), side,
                                  b.r_nodes, b.bases, keep, C.STEP2_FRACTION, levels=L, w1="haar")
    _assert_operators_equal(dt, ops, stats)


@pytest.mark.parametrize("chunk", [512, 1000])
def test_precompute_multi_chunk_emission_matches_oracle(lib, monkeypatch, chunk):
    """The emit -> scan -> rowptr path with several column chunks per row
    (the path every BASELINE operator is built through: C2 has 4 chunks, C3
    16): force 8 (512) and 5 uneven (1000) chunks at 64^2 and compare the whole
    operator with the oracle."""
    from paper_2203_12339_b200 import precompute as P
    from paper_2203_12339_b200.basis import build_basis
    from paper_2203_12339_b200.geometry import make_geometry_image

    monkeypatch.setattr(P, "EMIT_CHUNK", chunk)
    side, L, keep, K = 64, 3, 0.05, 8
    g = make_geometry_image(side, 10.0, 0.05, 8, 2203)
    b = build_basis(K, (8, 4))
    dt = P.precompute_compressed(g, b, L, keep, C.STEP2_FRACTION)
    ops = O.precompute_compressed(g.positions.astype(np.float64), g.area.astype(np.float64), side,
                                  b.r_nodes, b.bases, keep, C.STEP2_FRACTION, levels=L, w1="haar")
    _assert_operators_equal(dt, ops)


def test_c2_operator_matches_oracle_digests(lib, golden_dir):
    """BASELINE configs[1] (C2: 128^2, K = 8, 32 materials, L = 3, 5 %, 0.95):
    the GPU-built operator equals the oracle's, term by term: SHA-256 of
    cols / colptr / rowidx / f32 vals and the energy ledger
    (tests/golden/make_c2_digests.py ran the oracle here, ~11 min on a CPU
    core; the geometry image and basis travel as data)."""
    import hashlib
    import json

    from paper_2203_12339_b200.basis import DiffusionBasis
    from paper_2203_12339_b200.geometry import GeometryImage
    from paper_2203_12339_b200.precompute import precompute_compressed

    z = np.load(golden_dir / "c2_inputs.npz")
    want = json.loads((golden_dir / "c2_digests.json").read_text())
    side = int(z["side"])
    g = GeometryImage(side=side, positions=z["positions"], normals=z["normals"], area=z["area"])
    b = DiffusionBasis(r_nodes=z["r_nodes"], bases=z["bases"], singular_values=z["singular_values"],
                       sigma_nodes=z["sigma_nodes"], U=z["U"], eta=float(z["eta"]))
    dt = precompute_compressed(g, b, int(z["levels"]), float(z["step1_keep"]),
                               float(z["step2_fraction"]))

    def digest(a, dtype):
        return hashlib.sha256(np.ascontiguousarray(a, dtype=dtype).tobytes()).hexdigest()

    for k, (op, w) in enumerate(zip(dt.to_reference(), want["operators"])):
        assert op.nnz == w["nnz"] and op.cols.size == w["n_cols"], k
        assert digest(op.cols, "<u4") == w["cols"], k
        assert digest(op.colptr, "<i8") == w["colptr"], k
        assert digest(op.rowidx, "<u4") == w["rowidx"], k
        assert digest(op.vals.astype(np.float32), "<f4") == w["vals_f32"], k
        assert op.kept_energy == pytest.approx(w["kept_energy"], rel=1e-12)
        assert op.total_energy == pytest.approx(w["total_energy"], rel=1e-12)
        assert op.step1_entries == w["step1_entries"]


def test_step1_ties_flat_index(lib):
    """Exact ties in a row: the lowest flat indices win (wavelets.py:133-136)."""
    from paper_2203_12339_b200 import _lib
    from paper_2203_12339_b200.precompute import _tables

    side, L = 32, 2
    n = side * side
    f2t, t2f = _tables(side, L, "cuda")
    rng = np.random.default_rng(4)
    rows_flat = np.round(rng.standard_normal((8, n)), 1)
    rows_flat[0] = 1.5  # all equal
    D = torch.as_tensor(rows_flat[:, t2f.cpu().numpy()], device="cuda").contiguous()
    for n_keep in (1, 37, 500):
        u = torch.zeros(n // 32, dtype=torch.int32, device="cuda")
        _lib.call("sss_step1_select", _lib.ptr(D), n, 8, n_keep, _lib.ptr(t2f), _lib.ptr(u),
                  _lib.stream_ptr())
        want = np.zeros(n, bool)
        for r in rows_flat:
            want[O.compress_top_n(r, n_keep).indices] = True
        bits = np.unpackbits(u.cpu().numpy().view(np.uint8), bitorder="little").astype(bool)
        assert np.array_equal(bits, want)


def test_exact_mode_matches_projection_oracle(lib):
    """Exact mode (fp32 R_d x 64 materials, projected on U/S) vs the fp64
    exact-projection oracle: PCA transfer coefficients within 1e-3 of
    max |b_k| (BASELINE: "precompute PCA coefficients within 1e-3")."""
    from paper_2203_12339_b200.precompute import PairPass, _tables

    cfg = C.C5
    side, L = 32, 3
    g, b = _setup(cfg, side, amp=0.1)
    n = side * side
    pp = PairPass(g, b, L, exact=True)
    D = torch.empty((n, n), dtype=torch.float64, device="cuda")
    f2t, _ = _tables(side, L, "cuda")
    f2t = f2t.cpu().numpy()
    pos, area = g.positions.astype(np.float64), g.area.astype(np.float64)
    P = O.exact_projection_coeffs(b.U, b.singular_values, b.r_nodes, b.K)
    pts = np.random.default_rng(0).choice(n, 12, replace=False)
    ref = O.transfer_block_exact(pos[pts], pos, area, b.r_max, b.sigma_nodes, C.ETA, P)
    for k in range(b.K):
        pp.run(k, D, None)
        want = O.haar2d_fwd(ref[:, k].reshape(-1, side, side), L).reshape(len(pts), n)
        got = D.cpu().numpy()[_rows_tm(pts, side, L)][:, f2t]
        scale = np.abs(b.bases[k]).max() * area.max()
        assert np.abs(got - want).max() <= 1e-3 * scale, k


def test_kfused_exact_rows_equal_per_term_pass(lib):
    """The K-fused streamed exact pass (sss_pair_rows_exact: R_d once per pair,
    all K terms, constants folded per material) reproduces the per-term
    pass's step-1 rows (sss_pair_block exact mode) to fp32 rounding, block by
    block; its per-term unions agree up to near-tie columns; sampled rows are
    within 1e-3 of the fp64 projection oracle."""
    from paper_2203_12339_b200.precompute import PairPass, _tables, step1_unions_exact

    cfg = C.C5
    side, L = 32, 3
    g, b = _setup(cfg, side, amp=0.1)
    n, T2 = side * side, 64
    pp = PairPass(g, b, L, exact=True)
    f2t, t2f = _tables(side, L, "cuda")
    Dfull = torch.empty((n, n), dtype=torch.float64, device="cuda")
    nrt = 3
    Dblk = torch.empty((b.K, nrt * T2, n), dtype=torch.float64, device="cuda")
    rt0 = 5
    pp.run_rows_exact(rt0, nrt, Dblk)
    for k in range(b.K):
        pp.run(k, Dfull, None)
        want = Dfull[rt0 * T2:(rt0 + nrt) * T2]
        scale = want.abs().max().item()
        assert (Dblk[k] - want).abs().max().item() <= 1e-4 * scale, k
    keep = max(int(round(cfg.step1_keep * n)), 1)
    unions, _ = step1_unions_exact(pp, keep, t2f, block_bytes=8 * b.K * T2 * n * 5)  # 5-tile blocks
    for k in range(b.K):
        pp.run(k, Dfull, None)
        u = torch.zeros((n + 31) // 32, dtype=torch.int32, device="cuda")
        lib.sss_step1_select(Dfull.data_ptr(), n, n, keep, t2f.data_ptr(), u.data_ptr(), None)
        torch.cuda.synchronize()
        diff = (unions[k] ^ u).cpu().numpy().view(np.uint32)
        a = int(np.unpackbits(u.cpu().numpy().view(np.uint8)).sum())
        assert int(np.unpackbits(diff.view(np.uint8)).sum()) <= max(2, a // 200), k
    # against the fp64 projection oracle on sampled rows of one block
    pos, area = g.positions.astype(np.float64), g.area.astype(np.float64)
    P = O.exact_projection_coeffs(b.U, b.singular_values, b.r_nodes, b.K)
    f2t_h = f2t.cpu().numpy()
    rows_tm = np.arange(rt0 * T2, (rt0 + nrt) * T2)[::17]
    T, tpr = 1 << L, side >> L  # tile-major receiver row -> its grid point
    tile, loc = rows_tm // T2, rows_tm % T2
    pts = ((tile // tpr) * T + loc // T) * side + (tile % tpr) * T + loc % T
    ref = O.transfer_block_exact(pos[pts], pos, area, b.r_max, b.sigma_nodes, C.ETA, P)
    for k in range(b.K):
        want = O.haar2d_fwd(ref[:, k].reshape(-1, side, side), L).reshape(len(pts), n)
        got = Dblk[k].cpu().numpy()[rows_tm - rt0 * T2][:, f2t_h]
        assert np.abs(got - want).max() <= 1e-3 * np.abs(b.bases[k]).max() * area.max(), k
