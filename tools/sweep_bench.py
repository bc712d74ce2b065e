"""C4 (BASELINE configs[3]) batched material sweep on B200: 256^2 geometry
image, K=12, SH5 light, M=256 materials per RGB; times the tcgen05 sweep
contraction + shade (HBM-write-bound: 3 x M x N fp32 out) and the operand
preparation. Usage: python tools/sweep_bench.py [--side 256] [--reps 20]"""
import argparse
import json
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, b in ev:
        a.record()
        fn()
        b.record()
    torch.cuda.synchronize()
    return float(np.median([a.elapsed_time(b) for a, b in ev])) * 1e3


def measure(side=256, reps=20):
    """C4 sweep measurement dict (used by bench.py and main)."""
    from paper_2203_12339_b200 import _lib
    from paper_2203_12339_b200 import lighting as LT
    from paper_2203_12339_b200.basis import OpticalMaterial, build_basis
    from paper_2203_12339_b200.config import CONFIGS, SIGMA_BOX
    from paper_2203_12339_b200.geometry import make_geometry_image
    from paper_2203_12339_b200.precompute import precompute_compressed
    from paper_2203_12339_b200.runtime import Scene, SHLight

    _lib.load()
    cfg = CONFIGS["batched_sweep_256"].with_(side=side)
    M = cfg.extra["materials"]
    g = make_geometry_image(cfg.side, cfg.radius, cfg.bump_amp, cfg.bump_terms, cfg.seed)
    b = build_basis(cfg.K, cfg.lattice)
    dt = precompute_compressed(g, b, cfg.levels, cfg.step1_keep, cfg.step2_fraction)
    m0 = OpticalMaterial(sigma_s_prime=cfg.material[0], sigma_a=cfg.material[1], eta=cfg.material[2])
    sc = Scene(g, dt, b, m0, SHLight(LT.random_sh_light(cfg.sh_bands, 3)))
    sc.relight()
    rng = np.random.default_rng(4)
    lo_e, hi_e = cfg.extra["eta_range"]
    mats = [OpticalMaterial(sigma_s_prime=np.exp(rng.uniform(np.log(SIGMA_BOX[0]), np.log(SIGMA_BOX[1]), 3)),
                            sigma_a=np.exp(rng.uniform(np.log(SIGMA_BOX[2]), np.log(SIGMA_BOX[3]), 3)),
                            eta=float(rng.uniform(lo_e, hi_e))) for _ in range(M)]
    ops = sc.sweep_prepare(mats)
    out = torch.empty((3, M, sc.n), dtype=torch.float32, device="cuda")
    us_gemm = timed(lambda: sc.sweep_launch(ops, out), reps)
    us_prep = timed(lambda: sc.sweep_prepare(mats), max(3, reps // 4))
    out_bytes = out.numel() * 4
    in_bytes = 3 * sc.n * 16 * 2 + 3 * M * 16 * 2 + sc.n * 24 + M * 4
    peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"]
    res = {"config": cfg.name, "points": sc.n, "K": cfg.K, "materials": M,
           "sweep_gemm_us": us_gemm, "prepare_us_incl_host": us_prep,
           "out_bytes": out_bytes, "alg_bytes": out_bytes + in_bytes,
           "achieved_GBps": (out_bytes + in_bytes) / (us_gemm * 1e-6) / 1e9, "peak_GBps": peak,
           "frac": (out_bytes + in_bytes) / (us_gemm * 1e-6) / 1e9 / peak,
           "flops": 2 * 3 * sc.n * M * cfg.K,
           "radiance_points_per_s": 3 * M * sc.n / (us_gemm * 1e-6) / 3,
           "finite": bool(torch.isfinite(out).all()), "max": float(out.max())}
    del sc, dt, ops, out
    torch.cuda.empty_cache()
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--side", type=int, default=256)
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    print(json.dumps(measure(a.side, a.reps)))


if __name__ == "__main__":
    main()
