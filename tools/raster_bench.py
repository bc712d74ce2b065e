"""Raster stage timing: the C3 256^2 geometry-image mesh
(130050 triangles) rendered at 1280x720 with the bench camera, CUDA events
around the device launches (vertex colours + clear + 3 raster passes +
resolve/sRGB), and the whole render_image call with the u8 image copied to
the host; the oracle's raster_fill on the same inputs for scale.

    python tools/raster_bench.py [--side 256] [--width 1280] [--height 720]
"""

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--side", type=int, default=256)
    ap.add_argument("--width", type=int, default=1280)
    ap.add_argument("--height", type=int, default=720)
    ap.add_argument("--iters", type=int, default=50)
    ap.add_argument("--cpu", action="store_true", help="also time the oracle raster")
    a = ap.parse_args()
    from paper_2203_12339_b200.geometry import make_geometry_image
    from paper_2203_12339_b200.raster import Rasterizer, mesh_of
    from paper_2203_12339_b200.runtime import Camera

    geo = make_geometry_image(a.side)
    mesh = mesh_of(geo)
    rad = torch.rand((geo.count, 3), device="cuda", dtype=torch.float32)
    cam = Camera(position=np.array([60.0, 45.0, 150.0]), look_at=np.zeros(3), fov_y_degrees=10.0)
    r = Rasterizer(mesh, a.width, a.height)
    for _ in range(3):
        r.render(rad, cam)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(a.iters):
        r.set_radiance(rad)
        r.launch()
    e1.record()
    torch.cuda.synchronize()
    dev_ms = e0.elapsed_time(e1) / a.iters
    t0 = time.perf_counter()
    for _ in range(a.iters):
        img = r.render(rad, cam)
    e2e_ms = (time.perf_counter() - t0) * 1e3 / a.iters
    out = {"kernel": "raster (project + colours + depth/pick/resolve + sRGB)", "side": a.side,
           "triangles": int(mesh.triangles.shape[0]), "width": a.width, "height": a.height,
           "device_ms": dev_ms, "render_image_ms": e2e_ms,
           "covered_frac": float((img > 0).any(-1).mean())}
    if a.cpu:
        from oracle import sss_oracle as O

        t0 = time.perf_counter()
        O.render_image(mesh.vertices, mesh.triangles, np.arange(geo.count),
                       rad.cpu().numpy().astype(np.float64), cam.position, cam.look_at, cam.up,
                       cam.fov_y_degrees, a.width, a.height)
        out["oracle_ms"] = (time.perf_counter() - t0) * 1e3
    print(json.dumps(out))


if __name__ == "__main__":
    main()
