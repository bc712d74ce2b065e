"""Direct lights with shadow rays at 256^2 (C3 geometry): one point, one
directional and one sphere light (64 cone strata), timed on the GPU; rays/s.
Usage: python tools/direct_bench.py"""
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    from paper_2203_12339_b200 import _lib
    from paper_2203_12339_b200.config import CONFIGS
    from paper_2203_12339_b200.geometry import make_geometry_image
    from paper_2203_12339_b200.shadows import (DirectionalLight, LightRig, PointLight,
                                               SphereLight, build_bvh, grid_triangles)

    _lib.load()
    cfg = CONFIGS["env_large_256"]
    g = make_geometry_image(cfg.side, cfg.radius, cfg.bump_amp, cfg.bump_terms, cfg.seed)
    t0 = time.perf_counter()
    bvh = build_bvh(g.positions.astype(np.float64), grid_triangles(cfg.side))
    build_s = time.perf_counter() - t0
    d = lambda a, dt: torch.as_tensor(np.ascontiguousarray(a, dt), device="cuda")
    rig = LightRig(lights=(PointLight(position=[25.0, 18.0, 30.0], intensity=[900.0, 700.0, 500.0]),
                           DirectionalLight(direction=[-0.3, -1.0, -0.4], irradiance=[0.8, 0.9, 1.0]),
                           SphereLight(center=[-14.0, 6.0, 16.0], radius=3.0, radiance=[2.0, 1.5, 1.0])))
    n = g.count
    pos, nrm = d(g.positions, np.float32), d(g.normals, np.float32)
    mat = d(np.array([1, 1, 1, 0.01, 0.01, 0.01, 1.3]), np.float64)
    nodes, tris = bvh.packed()
    bufs = [d(nodes, np.float64), d(tris, np.float64)]
    out = {"points": n, "triangles": int(bvh.v0.shape[0]), "bvh_nodes": int(bvh.node_min.shape[0]),
           "bvh_build_s": build_s}
    import os
    cases = [(f"point_split{k}", rig.lights[:1], k) for k in range(5)]
    cases += [(f"directional_split{k}", rig.lights[1:2], k) for k in range(5)]
    cases += [("sphere64", rig.lights[2:], 3), ("all3", rig.lights, 3)]
    for name, lights, split in cases:
        os.environ["SSS_DIRECT_SPLIT"] = str(split)
        rig_l = LightRig(lights=lights)
        L = d(rig_l.packed(), np.float64)
        kinds = torch.tensor(rig_l.kinds())
        E = torch.empty((3, n), dtype=torch.float64, device="cuda")
        call = lambda: _lib.call("sss_direct_irradiance", n, _lib.ptr(pos), _lib.ptr(nrm), len(lights),
                                 _lib.ptr(kinds), _lib.ptr(L), _lib.ptr(mat), bvh.ray_offset,
                                 bvh.bbox_diagonal, *[_lib.ptr(b) for b in bufs], _lib.ptr(E),
                                 _lib.stream_ptr())
        call()
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ev[0].record()
        for _ in range(10):
            call()
        ev[1].record()
        torch.cuda.synchronize()
        us = ev[0].elapsed_time(ev[1]) / 10 * 1e3
        rays = n * (64 if name == "sphere64" else (66 if name == "all3" else 1))
        out[f"{name}_E_sum"] = float(E.sum())
        out[f"{name}_us"] = us
        out[f"{name}_rays_per_s_upper"] = rays / (us * 1e-6)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
