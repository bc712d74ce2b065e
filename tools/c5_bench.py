"""C5 (BASELINE configs[4]): the exact dipole pair pass at 256^2 — fp32 R_d
of all 65536^2 ordered pairs at 64 training materials, projected on K = 8
PCA terms, w0 Haar per row, per-row top 2 % (step 1 + per-term unions) —
K-fused and streamed by receiver-tile blocks (precompute.step1_unions_exact).

Reports pairs/s and the algorithmic FP32 rate (2.0 kFLOP + 256
MUFU per pair) against the FP32 peak (SMs x 128 x 2 x max SM clock).

    python tools/c5_bench.py [--side 256] [--reps 1]
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

FLOP_PER_PAIR = 2000.0   # SURVEY §8d, FFMA = 2 flops
MUFU_PER_PAIR = 256.0


def measure(side=256, reps=1):
    from paper_2203_12339_b200 import _lib
    from paper_2203_12339_b200.basis import build_basis
    from paper_2203_12339_b200.config import CONFIGS
    from paper_2203_12339_b200.geometry import make_geometry_image
    from paper_2203_12339_b200.precompute import PairPass, _tables, step1_unions_exact

    _lib.load()
    cfg = CONFIGS["dipole_precompute_256"].with_(side=side)
    g = make_geometry_image(cfg.side, cfg.radius, cfg.bump_amp, cfg.bump_terms, cfg.seed)
    b = build_basis(cfg.K, cfg.lattice)
    n = g.count
    pp = PairPass(g, b, cfg.levels, exact=True)
    _, t2f = _tables(cfg.side, cfg.levels, "cuda")
    keep = max(int(round(cfg.step1_keep * n)), 1)
    # warm-up on one block
    D = torch.empty((b.K, 64, n), dtype=torch.float64, device="cuda")
    pp.run_rows_exact(0, 1, D)
    del D
    torch.cuda.synchronize()
    best = None
    for _ in range(reps):
        st = {}
        t0 = time.perf_counter()
        unions, _ = step1_unions_exact(pp, keep, t2f, stats=st)
        torch.cuda.synchronize()
        st["wall_s"] = time.perf_counter() - t0
        if best is None or st["pair_s"] < best["pair_s"]:
            best = st
    props = torch.cuda.get_device_properties(0)
    peak = props.multi_processor_count * 128 * 2 * 1.965e9
    pairs = n * n
    out = {"config": cfg.name, "side": cfg.side, "pairs": pairs, "K": b.K,
           "materials": int(b.sigma_nodes.shape[0]), "block_receiver_tiles": best["block_tiles"],
           "pair_pass_s": best["pair_s"], "step1_select_s": best["select_s"],
           "step1_total_s": best["pair_s"] + best["select_s"], "wall_s": best["wall_s"],
           "pairs_per_s": pairs / best["pair_s"],
           "algorithmic_tflops": FLOP_PER_PAIR * pairs / best["pair_s"] / 1e12,
           "fp32_peak_tflops": peak / 1e12,
           "fp32_frac": FLOP_PER_PAIR * pairs / best["pair_s"] / peak,
           "mufu_per_s": MUFU_PER_PAIR * pairs / best["pair_s"],
           "union_sizes": [int(np.unpackbits(u.cpu().numpy().view(np.uint8)).sum()) for u in unions],
           "note": "K-fused: R_d evaluated once per pair for all K terms (was once per term)"}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--side", type=int, default=256)
    ap.add_argument("--reps", type=int, default=1)
    a = ap.parse_args()
    print(json.dumps(measure(a.side, a.reps)))


if __name__ == "__main__":
    main()
