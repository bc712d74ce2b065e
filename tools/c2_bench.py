"""C2 (BASELINE configs[1], medium interactive) on B200: 128^2 geometry image,
K=8 over 32 training materials, SH order 5, 3-level Haar, 5 % per row; every
frame applies a seeded uniform SO(3) rotation of the SH light and a new
log-uniform material. Device-timed relight + edit frames (CUDA graphs, the
light and material uploaded into the graph's device buffers), and the same
sequence through the public API (host SH coefficients in, FrameResult out).

    python tools/c2_bench.py [--frames 100]
"""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def measure(frames=100):
    from paper_2203_12339_b200 import _lib
    from paper_2203_12339_b200 import lighting as LT
    from paper_2203_12339_b200.basis import OpticalMaterial, build_basis
    from paper_2203_12339_b200.config import C2, SIGMA_BOX
    from paper_2203_12339_b200.geometry import from_config
    from paper_2203_12339_b200.precompute import precompute_compressed
    from paper_2203_12339_b200.runtime import Scene, SHLight

    _lib.load()
    g = from_config(C2)
    b = build_basis(C2.K, C2.lattice)
    t0 = time.perf_counter()
    dt = precompute_compressed(g, b, C2.levels, C2.step1_keep, C2.step2_fraction)
    torch.cuda.synchronize()
    pre_s = time.perf_counter() - t0
    rng = np.random.default_rng(2203)
    L0 = LT.random_sh_light(C2.sh_bands, 5)
    lights = [LT.rotate_sh(L0, LT.random_rotation(rng)) for _ in range(frames + 5)]

    def mat():
        lu = lambda lo, hi: np.exp(rng.uniform(np.log(lo), np.log(hi), 3))  # noqa: E731
        return OpticalMaterial(sigma_s_prime=lu(SIGMA_BOX[0], SIGMA_BOX[1]),
                               sigma_a=lu(SIGMA_BOX[2], SIGMA_BOX[3]), eta=C2.material[2])

    mats = [mat() for _ in range(frames + 5)]
    sc = Scene(g, dt, b, mats[0], SHLight(lights[0]))
    for f in range(3):
        sc.set_light(SHLight(lights[f]))
    sc.capture()
    dev_L = torch.as_tensor(np.stack(lights), device="cuda")
    dev_m = torch.as_tensor(np.stack([np.concatenate([m.sigma_s_prime, m.sigma_a, [m.eta]])
                                      for m in mats]), device="cuda")
    # each frame: new light (relight graph) and new material (edit graph)
    for f in range(5):
        sc.light_buf.copy_(dev_L[f])
        sc.replay(False)
        sc.material_buf.copy_(dev_m[f])
        sc.replay(True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for f in range(frames):
        sc.light_buf.copy_(dev_L[5 + f], non_blocking=True)
        sc.replay(False)
        sc.material_buf.copy_(dev_m[5 + f], non_blocking=True)
        sc.replay(True)
    e1.record()
    torch.cuda.synchronize()
    dev_ms = e0.elapsed_time(e1) / frames
    # public API: host SH light + host material in, FrameResult (numpy) out
    t0 = time.perf_counter()
    for f in range(frames):
        sc.set_light(SHLight(lights[5 + f]))
        sc.set_material(mats[5 + f])
    api_ms = (time.perf_counter() - t0) * 1e3 / frames
    n = g.count
    return {"config": C2.name, "points": n, "frames": frames, "operator_nnz": dt.nnz,
            "precompute_s": pre_s, "device_ms_per_frame": dev_ms,
            "device_points_per_s": n / (dev_ms / 1e3), "api_ms_per_frame": api_ms,
            "api_points_per_s": n / (api_ms / 1e3),
            "frame": "rotated SH light (relight) + new material (edit) per frame"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=100)
    a = ap.parse_args()
    print(json.dumps(measure(a.frames)))


if __name__ == "__main__":
    main()
