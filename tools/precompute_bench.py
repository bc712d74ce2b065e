"""C5 (BASELINE configs[4], dipole precompute 256^2) measurements: the pair
pass alone per PCA term (lerp and exact mode; pairs/s), and the whole GPU
precompute (pair pass -> step 1 -> step 2 -> emit, all K) in both modes.

    python tools/precompute_bench.py [--side 256] [--skip-full]
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


def measure(side=256, skip_full=False, ks=2):
    """C5 measurement dict (used by bench.py and main)."""
    from paper_2203_12339_b200 import _lib
    from paper_2203_12339_b200.basis import build_basis
    from paper_2203_12339_b200.config import CONFIGS
    from paper_2203_12339_b200.geometry import make_geometry_image
    from paper_2203_12339_b200.precompute import PairPass, precompute_compressed

    _lib.load()
    cfg = CONFIGS["dipole_precompute_256"].with_(side=side)
    g = make_geometry_image(cfg.side, cfg.radius, cfg.bump_amp, cfg.bump_terms, cfg.seed)
    b = build_basis(cfg.K, cfg.lattice)
    n = g.count
    out = {"config": cfg.name, "side": cfg.side, "points": n, "pairs": n * n, "K": cfg.K,
           "materials": int(np.prod(cfg.lattice))}
    D = torch.empty(n * n, dtype=torch.float64, device="cuda")
    M = torch.empty(n * n, dtype=torch.float64, device="cuda")
    for exact in (False, True):
        pp = PairPass(g, b, cfg.levels, exact=exact)
        pp.run(0, D, M)
        torch.cuda.synchronize()
        ms = []
        for k in range(ks):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            pp.run(k, D, M)
            e1.record()
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
        t = float(np.mean(ms)) / 1e3
        key = "exact" if exact else "lerp"
        out[f"pair_pass_{key}_s_per_k"] = t
        out[f"pair_pass_{key}_pairs_per_s_per_k"] = n * n / t
        # the reference evaluates all K terms per pair in one transfer_block
        out[f"pair_pass_{key}_pairs_per_s_all_K"] = n * n / (t * cfg.K)
        if exact:
            # per pair and term 64 x (2 rsqrt + 2 ex2) MUFU + ~24 FP32 ops
            mufu = n * n * out["materials"] * 4
            out["exact_mufu_per_s_per_k"] = mufu / t
    del D, M
    torch.cuda.empty_cache()
    if not skip_full:
        for exact in (False, True):
            st = {}
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            dt = precompute_compressed(g, b, cfg.levels, cfg.step1_keep, cfg.step2_fraction,
                                       exact=exact, stats=st)
            torch.cuda.synchronize()
            key = "exact" if exact else "lerp"
            out[f"precompute_{key}_s"] = time.perf_counter() - t0
            out[f"precompute_{key}_nnz"] = int(dt.nnz)
            del dt
            torch.cuda.empty_cache()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--side", type=int, default=256)
    ap.add_argument("--skip-full", action="store_true")
    ap.add_argument("--ks", type=int, default=2, help="PCA terms timed for the pair pass")
    a = ap.parse_args()
    print(json.dumps(measure(a.side, a.skip_full, a.ks)))


if __name__ == "__main__":
    main()
