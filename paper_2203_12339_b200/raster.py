"""Rasterisation of per-vertex radiance on the GPU.

Mirrors the reference's ``render_image`` / ``_project_vertices`` /
``raster_fill`` (runtime.py:230-273, _kernels_nb.py:316-359) and the service's
per-vertex frame payload (service.py:174-182), on top of the C ABI
(``sss_project_vertices``, ``sss_vertex_colors``, ``sss_raster_fill``,
``sss_encode_srgb8``). The linear image and the z-buffer are bitwise equal to
the reference's ``raster_fill`` on the same projected vertices.

``Rasterizer`` keeps the device buffers of one (mesh, width, height) so the
per-frame render is four launches and one u8 device-to-host copy;
``render_image`` is the reference-shaped one-shot call.
"""

from __future__ import annotations

import struct
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .geometry import GeometryImage
from .shadows import grid_triangles

FRAME_TAG = 1  # service.py:28


@dataclass(frozen=True)
class TriangleMesh:
    """surface.py:21-25 (vertices mm, unit normals, int triangles)."""

    vertices: np.ndarray  # (V, 3)
    normals: np.ndarray  # (V, 3)
    triangles: np.ndarray  # (T, 3)

    def content_hash(self) -> bytes:
        """surface.py:42-50: sha256 of float64 vertices, float64 normals and
        int32 triangles (what a container's mesh_hash records)."""
        import hashlib

        h = hashlib.sha256()
        h.update(np.ascontiguousarray(self.vertices, np.float64).tobytes())
        h.update(np.ascontiguousarray(self.normals, np.float64).tobytes())
        h.update(np.ascontiguousarray(self.triangles, np.int32).tobytes())
        return h.digest()


def mesh_of(geometry: GeometryImage) -> TriangleMesh:
    """The geometry image's grid triangulation; vertex i is surface sample i
    (so ``source_vertex`` is the identity)."""
    return TriangleMesh(geometry.positions.astype(np.float64),
                        geometry.normals.astype(np.float64),
                        grid_triangles(geometry.side))


def camera_frame(camera) -> np.ndarray:
    """(position, right, up, fwd) of _project_vertices (runtime.py:248-256)."""
    pos = np.asarray(camera.position, np.float64)
    fwd = np.asarray(camera.look_at, np.float64) - pos
    fwd = fwd / np.linalg.norm(fwd)
    right = np.cross(fwd, np.asarray(camera.up, np.float64))
    nr = np.linalg.norm(right)
    if nr < 1e-12:
        raise ValueError("camera up vector is parallel to the view direction")
    right /= nr
    up = np.cross(right, fwd)
    return np.concatenate([pos, right, up, fwd])


class Rasterizer:
    """Device-resident render target for one mesh and image size."""

    def __init__(self, mesh: TriangleMesh, width: int, height: int, source_vertex=None,
                 device=None):
        if width < 1 or height < 1:
            raise ValueError("image dimensions must be positive")
        _lib.load()
        dev = torch.device(device or "cuda")
        self.width, self.height = int(width), int(height)
        self.n_vertices = int(mesh.vertices.shape[0])
        self.n_tris = int(mesh.triangles.shape[0])
        f64 = dict(dtype=torch.float64, device=dev)
        self.vertices = torch.as_tensor(np.ascontiguousarray(mesh.vertices, np.float64), **f64)
        self.tris = torch.as_tensor(np.ascontiguousarray(mesh.triangles, np.int64), device=dev)
        self.source_vertex = (None if source_vertex is None else
                              torch.as_tensor(np.ascontiguousarray(source_vertex, np.int32),
                                              device=dev))
        n_pix = self.width * self.height
        self.proj = torch.empty((4, self.n_vertices), **f64)  # sx, sy, zn, iw
        self.colors = torch.zeros((self.n_vertices, 3), **f64)
        self.zbuf = torch.empty((self.height, self.width), **f64)
        self.img = torch.empty((self.height, self.width, 3), **f64)
        self.key = torch.empty(n_pix, dtype=torch.int64, device=dev)
        self.win = torch.empty(n_pix, dtype=torch.int32, device=dev)
        self.srgb = torch.empty((self.height, self.width, 3), dtype=torch.uint8, device=dev)
        self.cam = torch.empty(12, **f64)
        self._host = torch.empty((self.height, self.width, 3), dtype=torch.uint8, pin_memory=True)
        self._camera_key = None

    def set_camera(self, camera):
        key = (tuple(np.asarray(camera.position, float)), tuple(np.asarray(camera.look_at, float)),
               tuple(np.asarray(camera.up, float)), float(camera.fov_y_degrees))
        if key == self._camera_key:
            return
        self.cam.copy_(torch.as_tensor(camera_frame(camera)))
        f = 1.0 / np.tan(np.radians(camera.fov_y_degrees) / 2.0)
        sx, sy, zn, iw = self.proj
        _lib.call("sss_project_vertices", _lib.ptr(self.vertices), self.n_vertices,
                  _lib.ptr(self.cam), float(f), self.width / self.height, self.width, self.height,
                  _lib.ptr(sx), _lib.ptr(sy), _lib.ptr(zn), _lib.ptr(iw), _lib.stream_ptr())
        self._camera_key = key

    def set_radiance(self, radiance: torch.Tensor):
        """radiance (N, 3) f32 on the device (e.g. ``Scene.radiance``)."""
        rad = radiance.to(device=self.colors.device, dtype=torch.float32).contiguous()
        if self.source_vertex is None and rad.shape[0] != self.n_vertices:
            raise ValueError("radiance rows must match the mesh vertices")
        self.colors.zero_()
        _lib.call("sss_vertex_colors", _lib.ptr(rad), _lib.ptr(self.source_vertex),
                  int(rad.shape[0]), _lib.ptr(self.colors), _lib.stream_ptr())

    def launch(self, exposure: float = 1.0, background=(0.0, 0.0, 0.0)):
        """Clear, rasterise and encode on the current stream (no sync)."""
        b = np.broadcast_to(np.asarray(background, np.float64), (3,))
        _lib.call("sss_raster_clear", self.height, self.width, float(b[0]), float(b[1]),
                  float(b[2]), _lib.ptr(self.zbuf), _lib.ptr(self.img), _lib.stream_ptr())
        sx, sy, zn, iw = self.proj
        _lib.call("sss_raster_fill", _lib.ptr(self.tris), self.n_tris, _lib.ptr(sx), _lib.ptr(sy),
                  _lib.ptr(zn), _lib.ptr(iw), _lib.ptr(self.colors), self.height, self.width,
                  _lib.ptr(self.zbuf), _lib.ptr(self.img), _lib.ptr(self.key), _lib.ptr(self.win),
                  float(exposure), _lib.ptr(self.srgb), _lib.stream_ptr())

    def render(self, radiance: torch.Tensor, camera, exposure: float = 1.0,
               background=(0.0, 0.0, 0.0)) -> np.ndarray:
        self.set_camera(camera)
        self.set_radiance(radiance)
        self.launch(exposure, background)
        self._host.copy_(self.srgb, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        return self._host.numpy().copy()


def render_image(mesh: TriangleMesh, samples, frame, camera, width: int, height: int,
                 exposure: float = 1.0, background=(0.0, 0.0, 0.0)) -> np.ndarray:
    """runtime.py:230-245: Z-buffered rasterisation of per-vertex radiance to an
    sRGB u8 image (height, width, 3). ``samples`` supplies ``source_vertex``
    (None or a GeometryImage = identity); ``frame`` is a FrameResult (host
    radiance) or a device (N, 3) tensor."""
    if width < 1 or height < 1:
        raise ValueError("image dimensions must be positive")
    src = getattr(samples, "source_vertex", None)
    r = Rasterizer(mesh, width, height, source_vertex=src)
    rad = frame if isinstance(frame, torch.Tensor) else \
        torch.as_tensor(np.asarray(frame.radiance, np.float32))
    return r.render(rad, camera, exposure, background)


def frame_payload(radiance: torch.Tensor, sequence: int, fmt: str = "srgb8",
                  exposure: float = 1.0, n_vertices: int = None, source_vertex=None) -> bytes:
    """The service's binary frame (service.py:174-182): header
    <B tag, I sequence, I vertex count> followed by per-vertex colours as
    little-endian f16 ("f16") or sRGB-quantised u8 (anything else)."""
    rad = radiance.to(dtype=torch.float32).contiguous()
    nv = int(n_vertices if n_vertices is not None else rad.shape[0])
    colors = torch.zeros((nv, 3), dtype=torch.float64, device=rad.device)
    src = None if source_vertex is None else torch.as_tensor(
        np.ascontiguousarray(source_vertex, np.int32), device=rad.device)
    _lib.call("sss_vertex_colors", _lib.ptr(rad), _lib.ptr(src), int(rad.shape[0]),
              _lib.ptr(colors), _lib.stream_ptr())
    head = struct.pack("<BII", FRAME_TAG, int(sequence), nv)
    if fmt == "f16":
        return head + colors.to(torch.float16).cpu().numpy().astype("<f2").tobytes()
    out = torch.empty(nv * 3, dtype=torch.uint8, device=rad.device)
    _lib.call("sss_encode_srgb8", _lib.ptr(colors), nv * 3, float(exposure), _lib.ptr(out),
              _lib.stream_ptr())
    return head + out.cpu().numpy().tobytes()
