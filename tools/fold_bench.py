"""Visibility precompute + ambient folding timing at C3
(256^2 geometry image, K=8 operator from the GPU precompute), face side 16
(D = 1536 cubemap directions, 100.7 M shadow rays), and the per-frame cost
of a LightRig frame (point light + folded ambient environment) as a CUDA
graph replay, with and without the ambient term.

    python tools/fold_bench.py [--side 256] [--face-side 16]
"""

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--side", type=int, default=256)
    ap.add_argument("--face-side", type=int, default=16)
    ap.add_argument("--reps", type=int, default=50)
    a = ap.parse_args()
    from paper_2203_12339_b200 import config as C
    from paper_2203_12339_b200 import folding as F
    from paper_2203_12339_b200.basis import OpticalMaterial, build_basis
    from paper_2203_12339_b200.geometry import make_geometry_image
    from paper_2203_12339_b200.precompute import precompute_compressed
    from paper_2203_12339_b200.runtime import Scene
    from paper_2203_12339_b200.shadows import AmbientLight, LightRig, PointLight

    cfg = C.C3.with_(side=a.side)
    g = make_geometry_image(cfg.side, cfg.radius, cfg.bump_amp, cfg.bump_terms, cfg.seed)
    b = build_basis(cfg.K, cfg.lattice)
    dt = precompute_compressed(g, b, cfg.levels, cfg.step1_keep, cfg.step2_fraction)
    torch.cuda.synchronize()
    out = {"side": cfg.side, "K": cfg.K, "face_side": a.face_side,
           "directions": 6 * a.face_side ** 2, "rays": 6 * a.face_side ** 2 * g.count}
    vis = F.precompute_visibility(g, a.face_side)  # warm (BVH build + launch)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    vis = F.precompute_visibility(g, a.face_side)
    torch.cuda.synchronize()
    out["visibility_s"] = time.perf_counter() - t0
    out["visibility_rays_per_s"] = out["rays"] / out["visibility_s"]
    out["visible_frac"] = float(vis.vis.float().mean())
    t0 = time.perf_counter()
    folded = F.fold_visibility(dt, vis, g, cfg.material[2])
    torch.cuda.synchronize()
    out["fold_s"] = time.perf_counter() - t0
    out["folded_nnz"] = int(folded.rows.numel())
    gbase, _ = F.row_layout(folded)
    w = torch.diff(gbase) // 32
    out["ell_entries"] = int(gbase[-1])
    out["ell_group_width"] = {"max": int(w.max()), "mean": float(w.float().mean())}
    m0 = OpticalMaterial(sigma_s_prime=cfg.material[0], sigma_a=cfg.material[1], eta=cfg.material[2])
    rng = np.random.default_rng(3)
    amb = AmbientLight(np.exp(rng.standard_normal((6, a.face_side, a.face_side, 3))))
    pt = PointLight(position=[40.0, 30.0, 60.0], intensity=[3e3, 2.5e3, 2e3])
    for name, rig in (("point", LightRig((pt,))), ("point+ambient", LightRig((pt, amb)))):
        sc = Scene(g, dt, b, m0, rig, e_keep=cfg.e_keep, folded=folded)
        sc.relight()
        sc.capture()
        out[f"frame_ms[{name}]"] = timed(lambda: sc.replay(False), a.reps)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
