"""GPU parity for rasterisation: render_image /
_project_vertices / raster_fill (runtime.py:230-273, _kernels_nb.py:316-359)
and the service frame payload (service.py:174-182).

Bars: raster_fill's z-buffer and linear image bitwise against the reference's
own output (tests/golden/raster.npz) on the same projected vertices — depth
ties (duplicate triangles), reversed winding, clipped vertices and a partly
filled initial z-buffer included; the projection bitwise against the oracle's
ordered dot products; the full render (u8) bitwise against the oracle's
render_image; the reference tests' camera cases (deterministic, behind the
object = background only, object actually rendered).
"""

import struct

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


def _fill(g, prefix, tris, colors, zb0, img0):
    from paper_2203_12339_b200 import _lib

    d = lambda a: torch.as_tensor(np.ascontiguousarray(a)).cuda()  # noqa: E731
    h, w = zb0.shape
    zb, img = d(zb0), d(img0)
    key = torch.empty(h * w, dtype=torch.int64, device="cuda")
    win = torch.empty(h * w, dtype=torch.int32, device="cuda")
    t = d(np.asarray(tris, np.int64))
    sx, sy, zn, iw = (d(g[f"{prefix}_{n}"]) for n in ("sx", "sy", "zn", "iw"))
    c = d(colors)
    _lib.call("sss_raster_fill", _lib.ptr(t), int(t.shape[0]), _lib.ptr(sx), _lib.ptr(sy),
              _lib.ptr(zn), _lib.ptr(iw), _lib.ptr(c), h, w, _lib.ptr(zb), _lib.ptr(img),
              _lib.ptr(key), _lib.ptr(win), 1.0, None, _lib.stream_ptr())
    torch.cuda.synchronize()
    return zb.cpu().numpy(), img.cpu().numpy()


def test_raster_fill_bitwise_vs_reference(lib, golden):
    g = golden("raster")
    zb, img = _fill(g, "r", g["r_tris"], g["r_colors"], g["r_zbuf0"], g["r_img0"])
    assert np.array_equal(zb, g["r_zbuf"])
    assert np.array_equal(img, g["r_img"])


def test_mesh_raster_bitwise_vs_reference(lib, golden):
    g = golden("raster")
    for ci in range(2):
        zb0 = np.full((72, 96), np.inf)
        img0 = np.empty((72, 96, 3))
        img0[:] = (0.02, 0.02, 0.03)
        zb, img = _fill(g, f"c{ci}", g["m_tris"], g["m_radiance"], zb0, img0)
        assert np.array_equal(zb, g[f"c{ci}_zbuf"]), ci
        assert np.array_equal(img, g[f"c{ci}_img"]), ci


def _camera(pos, at, fov=40.0):
    from paper_2203_12339_b200.runtime import Camera

    return Camera(position=np.asarray(pos, float), look_at=np.asarray(at, float), fov_y_degrees=fov)


def test_render_image_bitwise_vs_oracle(lib, golden):
    from paper_2203_12339_b200.raster import Rasterizer, TriangleMesh, render_image

    g = golden("raster")
    mesh = TriangleMesh(g["m_vertices"], g["m_vertices"], g["m_tris"])
    rad32 = g["m_radiance"].astype(np.float32)
    for ci in range(2):
        cam = _camera(g[f"c{ci}_pos"], g[f"c{ci}_at"], float(g[f"c{ci}_fov"]))
        r = Rasterizer(mesh, 96, 72)
        r.set_camera(cam)
        torch.cuda.synchronize()
        sx, sy, zn, iw = O.project_vertices(g["m_vertices"], cam.position, cam.look_at, cam.up,
                                            cam.fov_y_degrees, 96, 72)
        got = r.proj.cpu().numpy()
        for a, b in zip(got, (sx, sy, zn, iw)):
            assert np.array_equal(a, b)
        u8 = render_image(mesh, None, torch.as_tensor(rad32).cuda(), cam, 96, 72, exposure=2.0,
                          background=(0.02, 0.02, 0.03))
        ref_u8, ref_img, _ = O.render_image(g["m_vertices"], g["m_tris"],
                                            np.arange(g["m_vertices"].shape[0]),
                                            rad32.astype(np.float64), cam.position, cam.look_at,
                                            cam.up, cam.fov_y_degrees, 96, 72, exposure=2.0,
                                            background=(0.02, 0.02, 0.03))
        assert np.array_equal(u8, ref_u8), ci
        assert np.array_equal(r.render(torch.as_tensor(rad32).cuda(), cam, 2.0, (0.02, 0.02, 0.03)),
                              ref_u8)
        assert np.array_equal(r.img.cpu().numpy(), ref_img), ci


def test_scene_render_cases(lib):
    """test_runtime.py:115-143: deterministic, behind-the-object background
    only, object actually rendered; plus the 64^2 frame against the oracle."""
    from paper_2203_12339_b200.geometry import make_geometry_image
    from paper_2203_12339_b200.raster import Rasterizer, mesh_of

    geo = make_geometry_image(64)
    mesh = mesh_of(geo)
    rng = np.random.default_rng(5)
    rad = torch.as_tensor(np.abs(rng.standard_normal((geo.count, 3))).astype(np.float32)).cuda()
    r = Rasterizer(mesh, 96, 72)
    cam = _camera([0.0, 0.0, 180.0], [0.0, 0.0, 0.0], 10.0)
    a = r.render(rad, cam, exposure=2.0)
    b = r.render(rad, cam, exposure=2.0)
    assert np.array_equal(a, b) and a.shape == (72, 96, 3)
    assert (a > 8).any()
    ref_u8, _, _ = O.render_image(mesh.vertices, mesh.triangles, np.arange(geo.count),
                                  rad.cpu().numpy().astype(np.float64), cam.position, cam.look_at,
                                  cam.up, cam.fov_y_degrees, 96, 72, exposure=2.0)
    assert np.array_equal(a, ref_u8)
    away = _camera([0.0, 0.0, 200.0], [0.0, 0.0, 400.0])
    r2 = Rasterizer(mesh, 64, 64)
    assert np.all(r2.render(rad, away) == 0)


def test_frame_payload(lib):
    from paper_2203_12339_b200.raster import frame_payload

    rng = np.random.default_rng(9)
    rad = np.abs(rng.standard_normal((300, 3))).astype(np.float32)
    src = rng.permutation(400)[:300]
    p = frame_payload(torch.as_tensor(rad).cuda(), 7, "srgb8", 1.5, n_vertices=400,
                      source_vertex=src)
    tag, seq, nv = struct.unpack("<BII", p[:9])
    assert (tag, seq, nv) == (1, 7, 400)
    colors = np.zeros((400, 3))
    colors[src] = rad
    assert p[9:] == O.encode_srgb8(colors, 1.5).tobytes()
    p16 = frame_payload(torch.as_tensor(rad).cuda(), 8, "f16", n_vertices=400, source_vertex=src)
    assert p16[9:] == colors.astype("<f2").tobytes()


def test_scene_render_image(lib):
    """Scene.render_image renders the frame's device radiance; equal to the
    reference-shaped render_image on the host FrameResult."""
    from paper_2203_12339_b200 import config as C
    from paper_2203_12339_b200 import lighting as LT
    from paper_2203_12339_b200.basis import OpticalMaterial, build_basis
    from paper_2203_12339_b200.geometry import make_geometry_image
    from paper_2203_12339_b200.precompute import precompute_compressed
    from paper_2203_12339_b200.raster import mesh_of, render_image
    from paper_2203_12339_b200.runtime import Scene, SHLight

    g = make_geometry_image(32)
    b = build_basis(4, (4, 4))
    dt = precompute_compressed(g, b, 2, 0.10, C.STEP2_FRACTION)
    m = OpticalMaterial(sigma_s_prime=C.C1.material[0], sigma_a=C.C1.material[1], eta=1.3)
    sc = Scene(g, dt, b, m, SHLight(LT.random_sh_light(3, 5)))
    sc.camera = _camera([0.0, 0.0, 180.0], [0.0, 0.0, 0.0], 10.0)
    fr = sc.relight()
    a = sc.render_image(128, 96, exposure=2.0)
    b2 = render_image(mesh_of(g), g, fr, sc.camera, 128, 96, exposure=2.0)
    assert np.array_equal(a, b2)
    assert (a > 8).any()
