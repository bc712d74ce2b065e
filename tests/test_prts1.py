"""PRTS1 bridge against a container written by the
reference's own writer (tests/golden/ref16.prts, made by
tests/golden/make_golden.py from the 16^2 reference precompute)."""

import io
from pathlib import Path

import numpy as np
import pytest

from paper_2203_12339_b200 import prts1
from paper_2203_12339_b200.transfer import DeviceTransfer

GOLD = Path(__file__).resolve().parent / "golden"


def _ref_ops(golden):
    g = golden("precompute16")
    tag = "k0.1_f0.95"
    K = sum(1 for k in g.files if k.startswith(f"{tag}_op") and k.endswith("_cols"))
    return g, [(g[f"{tag}_op{k}_cols"], g[f"{tag}_op{k}_colptr"], g[f"{tag}_op{k}_rowidx"],
                g[f"{tag}_op{k}_vals"], g[f"{tag}_op{k}_e"]) for k in range(K)]


def test_reads_reference_container(golden):
    c = prts1.load_prts1(GOLD / "ref16.prts")
    g, ops = _ref_ops(golden)
    assert c.sample_count == 256 and c.grid_side == 16 and c.is_identity_geometry_image()
    assert c.step1_keep == 0.1 and c.step2_fraction == 0.95
    assert len(c.operators) == len(ops)
    for op, (cols, colptr, rowidx, vals, e) in zip(c.operators, ops):
        assert np.array_equal(op.cols, cols)
        assert np.array_equal(op.colptr, colptr)
        assert np.array_equal(op.rowidx, rowidx)
        assert np.array_equal(op.vals, vals.astype(np.float32).astype(np.float64))
        assert (op.kept_energy, op.total_energy, op.step1_entries) == (e[0], e[1], int(e[2]))
    b = golden("basis")
    assert np.array_equal(c.basis.r_nodes, b["r_nodes"])
    assert np.array_equal(c.basis.bases, b["4x4_K4_bases"])
    assert c.metadata["source"] == "sssrelight reference"


def test_writer_reproduces_reference_bytes(tmp_path):
    c = prts1.load_prts1(GOLD / "ref16.prts")
    out = tmp_path / "ours.prts"
    prts1.save_prts1(out, c.basis, c.operators, c.step1_keep, c.step2_fraction, c.grid_side,
                     mesh_hash=c.mesh_hash, metadata=c.metadata)
    assert out.read_bytes() == (GOLD / "ref16.prts").read_bytes()


def test_device_layout_round_trip_through_container(tmp_path):
    """reference container -> GPU frame layout (host tensors) -> back to
    reference operators -> PRTS1 -> identical operators."""
    c = prts1.load_prts1(GOLD / "ref16.prts")
    dt = prts1.to_device(c, levels=2, device="cpu")
    back = dt.to_reference()
    out = tmp_path / "rt.prts"
    prts1.save_prts1(out, c.basis, back, c.step1_keep, c.step2_fraction, 16,
                     mesh_hash=c.mesh_hash)
    c2 = prts1.load_prts1(out)
    for a, b in zip(c.operators, c2.operators):
        keep = np.diff(a.colptr) > 0
        assert np.array_equal(a.cols[keep], b.cols)
        assert np.array_equal(a.rowidx, b.rowidx)
        assert np.array_equal(a.vals, b.vals)


def test_rejects_bad_containers(tmp_path):
    data = (GOLD / "ref16.prts").read_bytes()
    bad = tmp_path / "bad.prts"
    bad.write_bytes(b"NOTPRTS1" + data[8:])
    with pytest.raises(prts1.PRTS1Error, match="not a PRTS1"):
        prts1.load_prts1(bad)
    bad.write_bytes(data[: len(data) // 2])
    with pytest.raises(prts1.PRTS1Error, match="truncated"):
        prts1.load_prts1(bad)
    with pytest.raises(prts1.PRTS1Error, match="different mesh"):
        prts1.load_prts1(GOLD / "ref16.prts", expected_mesh_hash=b"\0" * 32)


def test_default_mesh_hash_is_the_reference_content_hash(tmp_path):
    """save_prts1 without an explicit hash records TriangleMesh.content_hash
    (surface.py:42-50) of the geometry image's grid mesh, so the reference's
    Scene accepts the container for that mesh (runtime.py:72-73)."""
    import sys
    from pathlib import Path

    from paper_2203_12339_b200.geometry import make_geometry_image
    from paper_2203_12339_b200.shadows import grid_triangles

    c = prts1.load_prts1(GOLD / "ref16.prts")
    gi = make_geometry_image(16, amp=0.05, seed=11)
    out = tmp_path / "h.prts"
    prts1.save_prts1(out, c.basis, c.operators, c.step1_keep, c.step2_fraction, 16,
                     positions=gi.positions, normals=gi.normals)
    got = prts1.load_prts1(out).mesh_hash
    ref = Path(__file__).resolve().parents[1] / "baseline" / "_ref"
    if not (ref / "sssrelight").exists():
        pytest.skip("baseline/_ref not installed")
    sys.path.insert(0, str(ref))
    try:
        from sssrelight.surface import TriangleMesh
    finally:
        sys.path.remove(str(ref))
    mesh = TriangleMesh(vertices=gi.positions.astype(np.float64),
                        normals=gi.normals.astype(np.float64), triangles=grid_triangles(16))
    assert got == mesh.content_hash()


def test_gpu_layout_sidecar_round_trip(tmp_path):
    """The kfr frame layout of a reference container's operators, saved as a
    sidecar tied to the operators' digest, loads back identical; a digest of
    other operators is rejected (CPU: the layout build runs with torch)."""
    import torch

    from paper_2203_12339_b200.layout import kfr_layout, kfr_reference_apply

    c = prts1.load_prts1(GOLD / "ref16.prts")
    dt = prts1.to_device(c, levels=2, device="cpu")
    lay = kfr_layout(dt, chunk=64)
    dig = prts1.operators_digest(c.operators)
    side = tmp_path / "ref16.prts.kfr"
    prts1.save_gpu_layout(side, lay, dig)
    back = prts1.load_gpu_layout(side, dig, device="cpu")
    for k in ("items", "lane_len", "lane_dst", "batch_off", "stream", "partial_row", "multi_info"):
        assert torch.equal(getattr(back, k), getattr(lay, k)), k
    assert back.stats == lay.stats and back.n_items == lay.n_items
    x = torch.as_tensor(np.random.default_rng(1).standard_normal((3, dt.n)))
    assert torch.equal(kfr_reference_apply(back, x), kfr_reference_apply(lay, x))
    with pytest.raises(prts1.PRTS1Error):
        prts1.load_gpu_layout(side, "0" * 64, device="cpu")
