"""Generate golden fixtures by running the REAL reference (sssrelight).

Run in the build container only (the reference is not on the GPU box):

    python tests/golden/make_golden.py [--ref baseline/_ref]

The reference is imported from a writable copy (``pip install --no-deps
--target baseline/_ref /tmp/refpkg``; importing /root/reference in place would
write numba caches into it). ``SSSRELIGHT_NO_NUMBA=1`` selects the
numpy twin, which the reference's own tests assert is bitwise equal to the
numba kernels (tests/test_kernels.py:21-109).

Every fixture is small (kilobytes to ~1 MB) and is consumed by
``tests/test_oracle_golden.py``.
"""

from __future__ import annotations

import argparse
import os
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]


def _import_reference(path):
    os.environ.setdefault("SSSRELIGHT_NO_NUMBA", "1")
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_golden")
    sys.path.insert(0, str(path))
    import sssrelight  # noqa: F401
    return sssrelight


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", default=str(ROOT / "baseline" / "_ref"))
    ap.add_argument("--only", default=None, help="write just this fixture (e.g. raster)")
    args = ap.parse_args()
    _import_reference(args.ref)
    sys.path.insert(0, str(ROOT))
    if args.only == "raster":
        raster_fixture()
        return

    from sssrelight import _kernels_np as knp
    from sssrelight import basisgen as bg
    from sssrelight import dipole as dp
    from sssrelight import envmap as em
    from sssrelight import lighting as lt
    from sssrelight import transfer as tr
    from sssrelight import wavelets as wv
    from sssrelight.surface import QuadtreeAtlas, SurfaceSamples

    from paper_2203_12339_b200 import config as cfgs
    from paper_2203_12339_b200.geometry import make_geometry_image

    rng = np.random.default_rng(2203)

    # 1. wavelets: full pyramid via the reference kernels; L-level via the
    #    reference's own per-axis primitives in its level loop
    x = rng.standard_normal((4, 32, 32))
    out = dict(x=x, haar_fwd=knp.haar2d_fwd_batch(x), haar_inv=knp.haar2d_inv_batch(x),
               cdf_fwd=knp.cdf97_fwd_batch(x), cdf_inv=knp.cdf97_inv_batch(x))
    for L in (1, 2, 3):
        f = np.array(x, copy=True)
        s = 32
        for _ in range(L):
            sub = f[:, :s, :s]
            knp._haar_axis_fwd(sub)
            knp._haar_axis_fwd(sub.swapaxes(-1, -2))
            s //= 2
        out[f"haar_fwd_L{L}"] = f
        g = np.array(x, copy=True)
        s = 32 >> (L - 1)
        while s <= 32:
            sub = g[:, :s, :s]
            knp._haar_axis_inv(sub.swapaxes(-1, -2))
            knp._haar_axis_inv(sub)
            s *= 2
        out[f"haar_inv_L{L}"] = g
    np.savez_compressed(HERE / "wavelets.npz", **out)

    # 2. selection (ties included)
    v = np.round(rng.standard_normal(4096) * 4) / 4  # many exact ties
    sel = dict(v=v)
    for n in (0, 1, 7, 410, 1024, 4096):
        s = wv.compress_top_n(v, n)
        sel[f"top_{n}_idx"] = s.indices
        sel[f"top_{n}_val"] = s.values
        sel[f"top_{n}_e"] = np.array([s.total_energy, s.kept_energy])
    for f in (0.0, 0.5, 0.9, 0.95, 0.9999, 1.0):
        s = wv.compress_energy(v, f)
        sel[f"en_{f}_idx"] = s.indices
        sel[f"en_{f}_e"] = np.array([s.total_energy, s.kept_energy])
    np.savez_compressed(HERE / "select.npz", **sel)

    # 3. dipole physics
    pts = np.stack([rng.uniform(0.1, 10.0, 64), rng.uniform(0.001, 1.0, 64),
                    rng.uniform(1.0, 2.0, 64), rng.uniform(0.0, 50.0, 64)], axis=1)
    rd = np.array([dp.eval_rd(dp.derive_dipole_raw(a, b, c), r) for a, b, c, r in pts])
    cosv = np.linspace(0.0, 1.0, 33)
    ft = np.stack([dp.fresnel_transmittance(e, cosv) for e in (1.0, 1.2, 1.3, 1.5)])
    np.savez_compressed(HERE / "dipole.npz", pts=pts, rd=rd, cos=cosv, ft=ft,
                        fdr=np.array([dp.fdr(e) for e in (1.0, 1.2, 1.3, 1.5)]))

    # 4. PCA bases per config lattice (shipped as data)
    basis_out = {}
    for cfg in (cfgs.C1, cfgs.C2, cfgs.C4, cfgs.C5):
        grid0 = bg.build_sample_grid(bg.GridConfig(sigma_box=cfgs.SIGMA_BOX, eta=cfgs.ETA,
                                                   n_r=cfgs.N_R, sigma_lattice=2))
        sp = np.geomspace(cfgs.SIGMA_BOX[0], cfgs.SIGMA_BOX[1], cfg.lattice[0])
        sa = np.geomspace(cfgs.SIGMA_BOX[2], cfgs.SIGMA_BOX[3], cfg.lattice[1])
        nodes = np.stack(np.meshgrid(sp, sa, indexing="ij"), axis=-1).reshape(-1, 2)
        grid = bg.SampleGrid(r_nodes=grid0.r_nodes, sigma_nodes=nodes, eta=cfgs.ETA,
                             g=0.0, sigma_box=cfgs.SIGMA_BOX)
        basis = bg.decompose(bg.assemble_matrix(grid), cfg.K)
        mat = dp.OpticalMaterial(sigma_s_prime=cfg.material[0], sigma_a=cfg.material[1],
                                 eta=cfg.material[2])
        key = f"{cfg.lattice[0]}x{cfg.lattice[1]}_K{cfg.K}"
        basis_out[f"{key}_bases"] = basis.bases
        basis_out[f"{key}_sv"] = basis.singular_values
        basis_out[f"{key}_s"] = bg.project_material(basis, mat).s
        basis_out["r_nodes"] = grid.r_nodes
    np.savez_compressed(HERE / "basis.npz", **basis_out)

    # 5. transfer rows + CSC apply (test_kernels.py:31-91 shapes)
    n, k, nr = 200, 6, 64
    positions = rng.random((n, 3)) * 40.0
    areas = rng.random(n) + 0.1
    r_nodes = np.concatenate([[0.0], np.sort(rng.random(nr - 1)) * 60.0])
    bases = rng.standard_normal((k, nr))
    slopes = (bases[:, 1:] - bases[:, :-1]) / np.diff(r_nodes)
    rows = knp.transfer_block(positions[:8], positions, areas, r_nodes, bases, slopes)
    n_cols, out_len = 50, 512
    cols = np.sort(rng.choice(1024, n_cols, replace=False)).astype(np.uint32)
    counts = rng.integers(0, 20, n_cols)
    colptr = np.zeros(n_cols + 1, np.int64)
    colptr[1:] = np.cumsum(counts)
    rowidx = rng.integers(0, out_len, int(colptr[-1])).astype(np.uint32)
    vals = rng.standard_normal(int(colptr[-1]))
    x_idx = np.sort(rng.choice(1024, 100, replace=False)).astype(np.uint32)
    x_val = rng.standard_normal(100)
    csc_out = knp.csc_apply(cols, colptr, rowidx, vals, x_idx, x_val, out_len)
    np.savez_compressed(HERE / "kernels.npz", positions=positions, areas=areas,
                        r_nodes=r_nodes, bases=bases, rows=rows, cols=cols,
                        colptr=colptr, rowidx=rowidx, vals=vals, x_idx=x_idx,
                        x_val=x_val, csc_out=csc_out)

    # 6. the reference's full two-step precompute + a frame on a 16x16
    #    geometry image (identity atlas), full-pyramid Haar w0 + 9/7 w1
    side = 16
    gi = make_geometry_image(side, amp=0.05, seed=11)
    samples = SurfaceSamples(positions=gi.positions.astype(np.float64),
                             normals=gi.normals.astype(np.float64),
                             area=gi.area.astype(np.float64),
                             source_vertex=np.arange(side * side, dtype=np.int32))
    atlas = QuadtreeAtlas(part_count=1, grid_side=side,
                          part_of=np.zeros(side * side, np.uint32),
                          cell_of=np.arange(side * side, dtype=np.uint32),
                          inverse=np.arange(side * side, dtype=np.uint32).reshape(1, side, side))
    key = "4x4_K4"
    basis = bg.DiffusionBasis(r_nodes=basis_out["r_nodes"], bases=basis_out[f"{key}_bases"],
                              singular_values=basis_out[f"{key}_sv"], eta=cfgs.ETA, g=0.0,
                              sigma_box=cfgs.SIGMA_BOX)
    pre = {}
    for keep, frac in ((0.1, 0.95), (0.1, 0.9999)):
        ct = tr.precompute_compressed(samples, atlas, basis, keep, frac, spill_dir="/tmp")
        for ki, op in enumerate(ct.operators):
            tag = f"k{keep}_f{frac}_op{ki}"
            pre[f"{tag}_cols"] = op.cols
            pre[f"{tag}_colptr"] = op.colptr
            pre[f"{tag}_rowidx"] = op.rowidx
            pre[f"{tag}_vals"] = op.vals
            pre[f"{tag}_e"] = np.array([op.kept_energy, op.total_energy, op.step1_entries])
    # frame (runtime.py:109-216 composed from the reference's functions)
    ct = tr.precompute_compressed(samples, atlas, basis, 0.1, 0.95, spill_dir="/tmp")
    flat = tr.atlas_flat_cells(atlas)
    E = np.abs(rng.standard_normal((side * side, 3))) + 0.5
    mat = dp.OpticalMaterial(sigma_s_prime=cfgs.C1.material[0], sigma_a=cfgs.C1.material[1],
                             eta=cfgs.C1.material[2])
    keep = max(1, int(round(0.25 * side * side)))
    spectra = [wv.compress_top_n(tr.w0_forward(atlas, E[:, c], flat), keep) for c in range(3)]
    vk = np.zeros((basis.K, 3, side * side))
    for ki, op in enumerate(ct.operators):
        for c in range(3):
            vk[ki, c] = op.apply(spectra[c].indices, spectra[c].values, side * side)
    s = bg.project_material(basis, mat).s
    summed = np.einsum("ck,kcd->cd", s, vk)
    scatter = np.stack([tr.w1_inverse(atlas, summed[c], flat) for c in range(3)], axis=1)
    cam = np.array([0.0, 0.0, 180.0])
    view = cam[None, :] - samples.positions
    view /= np.linalg.norm(view, axis=1, keepdims=True)
    cos = np.clip(np.einsum("ij,ij->i", samples.normals, view), 0.0, 1.0)
    unclamped = scatter * (dp.fresnel_transmittance(mat.eta, cos) / np.pi)[:, None]
    pre.update(side=np.array(side), E=E, vk=vk, s=s, scatter=scatter, unclamped=unclamped,
               **{f"E_idx{c}": spectra[c].indices for c in range(3)})
    np.savez_compressed(HERE / "precompute16.npz", **pre)

    # 6b. the same operators + basis + identity atlas written by the
    #     reference's PRTS1 writer (container.py:81-137): the bridge fixture
    from sssrelight import container as ctn
    import hashlib

    mesh_hash = hashlib.sha256(np.ascontiguousarray(samples.positions).tobytes()).digest()
    ctn.save_container(HERE / "ref16.prts", basis, atlas, ct, mesh_hash,
                       metadata={"source": "sssrelight reference", "side": side})

    # 6c. direct lights with shadow rays on the geometry image's grid mesh
    #     (lighting.py:101-290): the reference's BVH any-hit and
    #     irradiance_direct for a point, a directional and a sphere light
    from sssrelight.surface import TriangleMesh
    from oracle import sss_oracle as O

    dside = 16
    dg = make_geometry_image(dside, amp=0.2, seed=5)
    dpos = dg.positions.astype(np.float64)
    dnrm = dg.normals.astype(np.float64)
    tris = O.grid_triangles(dside)
    mesh = TriangleMesh(vertices=dpos, normals=dnrm, triangles=tris)
    dsamples = SurfaceSamples(positions=dpos, normals=dnrm, area=dg.area.astype(np.float64),
                              source_vertex=np.arange(dside * dside, dtype=np.int32))
    accel = lt.RayAccelerator(mesh)
    lights = [lt.PointLight(position=[25.0, 18.0, 30.0], intensity=[900.0, 700.0, 500.0]),
              lt.DirectionalLight(direction=[-0.3, -1.0, -0.4], irradiance=[0.8, 0.9, 1.0]),
              lt.SphereLight(center=[-14.0, 6.0, 16.0], radius=3.0, radiance=[2.0, 1.5, 1.0])]
    rig = lt.LightRig(lights=tuple(lights))
    E_direct = lt.irradiance_direct(dsamples, rig, accel, 1.3)
    drng = np.random.default_rng(9)
    ro = dpos + accel.ray_offset * dnrm
    rd = drng.standard_normal((dside * dside, 3))
    rd /= np.linalg.norm(rd, axis=1, keepdims=True)
    rt = np.full(dside * dside, 50.0)
    hits = accel.any_hit(ro, rd, rt)
    np.savez_compressed(HERE / "direct.npz", side=np.array(dside), positions=dpos, normals=dnrm,
                        triangles=tris, E=E_direct, ray_o=ro, ray_d=rd, ray_t=rt, hits=hits,
                        eta=np.array(1.3), ray_offset=np.array(accel.ray_offset),
                        p_pos=lights[0].position, p_int=lights[0].intensity,
                        d_dir=lights[1].direction, d_irr=lights[1].irradiance,
                        s_c=lights[2].center, s_r=np.array(lights[2].radius),
                        s_rad=lights[2].radiance)

    # 6d. visibility precompute + ambient folding (transfer.py:368-451) on the
    #     self-occluding direct-light geometry: reference-built operators,
    #     binary visibility (face side 4: 96 directions), folded operators at
    #     the default fraction, and the folded ambient v_k of one environment
    fct = tr.precompute_compressed(dsamples, atlas, basis, 0.1, 0.95, spill_dir="/tmp")
    fvis = tr.precompute_visibility(dsamples, accel, face_side=4)
    fold = tr.fold_visibility(fct, fvis, dsamples, atlas, eta=1.3, fraction=0.9999)
    frng = np.random.default_rng(13)
    fenv = em.Cubemap(faces=frng.random((6, 4, 4, 3)) + 0.1)
    fspec = lt.project_environment(fenv, 32)
    fvk = np.zeros((basis.K, 3, dside * dside))
    for ki, op in enumerate(fold.operators):
        for c in range(3):
            fvk[ki, c] = op.apply(fspec[c].indices, fspec[c].values, dside * dside)
    fo = dict(side=np.array(dside), face_side=np.array(4), eta=np.array(1.3),
              fraction=np.array(0.9999), vis=fvis.matrix.astype(np.uint8), faces=fenv.faces,
              vk=fvk)
    for c in range(3):
        fo[f"env_idx{c}"] = fspec[c].indices
        fo[f"env_val{c}"] = fspec[c].values
    for tag, opl in (("op", fct.operators), ("fold", fold.operators)):
        for ki, op in enumerate(opl):
            fo[f"{tag}{ki}_cols"] = op.cols
            fo[f"{tag}{ki}_colptr"] = op.colptr
            fo[f"{tag}{ki}_rowidx"] = op.rowidx
            fo[f"{tag}{ki}_vals"] = op.vals
            fo[f"{tag}{ki}_e"] = np.array([op.kept_energy, op.total_energy, op.step1_entries])
    np.savez_compressed(HERE / "fold.npz", **fo)

    # 7. environment light: project_environment + dense ambient irradiance
    env_side = 8
    faces = np.exp(rng.standard_normal((6, env_side, env_side, 3)))
    cube = em.Cubemap(faces=faces)
    spectra = lt.project_environment(cube, 32)
    W = lt.visibility_weights(samples, np.ones((side * side, 6 * env_side ** 2)), env_side, 1.0)
    e_env = lt.ambient_irradiance_dense(samples, W,
                                        lt.reconstruct_environment(spectra, env_side))
    env = dict(faces=faces, W=W, E=e_env,
               dirs=em.face_directions(env_side), dom=em.face_solid_angles(env_side))
    for c in range(3):
        env[f"idx{c}"] = spectra[c].indices
        env[f"val{c}"] = spectra[c].values
    np.savez_compressed(HERE / "env.npz", **env)
    print("golden fixtures written to", HERE)
    raster_fixture()


def raster_fixture():
    """8. rasterisation: the reference's raster_fill on random triangles (the
    test_kernels.py:91-109 pattern plus duplicate / reversed triangles for
    depth ties and a partly filled initial z-buffer) and render_image's
    stages on a 16^2 geometry-image mesh (_project_vertices -> raster_fill ->
    linear_to_srgb), runtime.py:230-273."""
    from sssrelight import _kernels_np as knp
    from sssrelight import runtime as rt
    from sssrelight.envmap import linear_to_srgb

    from paper_2203_12339_b200.geometry import make_geometry_image
    from paper_2203_12339_b200.shadows import grid_triangles

    rng = np.random.default_rng(2271)
    out = {}
    n_tris, h, w = 60, 48, 64
    nv = 3 * n_tris
    tris = np.arange(nv, dtype=np.int64).reshape(n_tris, 3)
    tris[40:50] = tris[0:10]            # exact duplicates: equal depth, first wins
    tris[50:55] = tris[10:15][:, ::-1]  # reversed winding of earlier triangles
    sx = rng.uniform(-10, 74, nv)
    sy = rng.uniform(-10, 58, nv)
    zn = rng.uniform(0.5, 5.0, nv)
    iw = rng.uniform(0.2, 2.0, nv)
    iw[rng.random(nv) < 0.1] = 0.0
    colors = rng.random((nv, 3))
    zb = np.full((h, w), np.inf)
    zb[rng.random((h, w)) < 0.2] = 2.0   # pre-existing depth
    img = rng.random((h, w, 3))
    out.update(r_tris=tris, r_sx=sx, r_sy=sy, r_zn=zn, r_iw=iw, r_colors=colors,
               r_zbuf0=zb.copy(), r_img0=img.copy())
    knp.raster_fill(tris, sx, sy, zn, iw, colors, zb, img)
    out.update(r_zbuf=zb, r_img=img)

    g = make_geometry_image(16)
    verts = g.positions.astype(np.float64)
    gt = grid_triangles(16).astype(np.int64)
    rad = np.abs(rng.standard_normal((verts.shape[0], 3))).astype(np.float32).astype(np.float64)
    out.update(m_vertices=verts, m_tris=gt, m_radiance=rad)
    cams = [dict(position=[0.0, 0.0, 180.0], look_at=[0.0, 0.0, 0.0], fov_y_degrees=8.0),
            dict(position=[60.0, 45.0, 150.0], look_at=[0.0, 0.0, 0.0], fov_y_degrees=10.0)]
    for ci, cam in enumerate(cams):
        camera = rt.Camera(**cam)
        W, H = 96, 72
        sx, sy, zn, iw = rt._project_vertices(verts, camera, W, H)
        zb = np.full((H, W), np.inf)
        img = np.empty((H, W, 3))
        img[:] = (0.02, 0.02, 0.03)
        knp.raster_fill(gt, sx, sy, zn, iw, np.ascontiguousarray(rad), zb, img)
        u8 = (linear_to_srgb(img * 2.0) * 255.0 + 0.5).astype(np.uint8)
        out.update({f"c{ci}_pos": np.array(cam["position"]), f"c{ci}_at": np.array(cam["look_at"]),
                    f"c{ci}_fov": np.array(cam["fov_y_degrees"]), f"c{ci}_sx": sx,
                    f"c{ci}_sy": sy, f"c{ci}_zn": zn, f"c{ci}_iw": iw, f"c{ci}_img": img,
                    f"c{ci}_zbuf": zb, f"c{ci}_u8": u8})
    np.savez_compressed(HERE / "raster.npz", **out)
    print("raster fixture written")


if __name__ == "__main__":
    main()
