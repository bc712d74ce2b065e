"""Column working set of receiver regions on the C3 operator: rows grouped by
B x B blocks of 8x8 receiver tiles; distinct columns (union over rows and k)
per region, and the same restricted to columns kept in a frame.
Usage: python tools/region_cols.py"""
import json
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import bench as B
    from paper_2203_12339_b200 import _lib
    from paper_2203_12339_b200.config import CONFIGS

    _lib.load()
    cfg = CONFIGS["env_large_256"]
    g, b, dt, env, sc = B.setup_scene(cfg, 0, torch, {})
    sc.relight()
    n, K, L = dt.n, dt.K, dt.levels
    T2 = (1 << L) ** 2
    tpr = dt.side >> L
    rp = dt.rowptr.to(torch.int64)
    lens = (rp[:, 1:] - rp[:, :-1]).reshape(-1)
    base = int(rp[0, 0])
    tot = int(lens.sum())
    kr = torch.arange(K * n, device="cuda")
    row = torch.repeat_interleave(kr % n, lens)
    col = dt.cols[base:base + tot].to(torch.int64) & 0xFFFFFFFF
    kept = (sc.x != 0).any(dim=0)
    out = {}
    tile = row // T2
    tr, tc = tile // tpr, tile % tpr
    for Bk in (1, 2, 4):
        reg = (tr // Bk) * (tpr // Bk) + (tc // Bk)
        key = torch.unique(reg * n + col)
        per = torch.bincount(key // n)
        kk = torch.unique(reg[kept[col]] * n + col[kept[col]])
        perk = torch.bincount(kk // n)
        q = torch.quantile(per.float(), torch.tensor([0.5, 0.9, 0.99], device="cuda")).tolist()
        out[f"block{Bk}x{Bk}_tiles_quantiles_50_90_99"] = q
        out[f"block{Bk}x{Bk}_tiles"] = {
            "regions": int(per.numel()), "rows_per_region": Bk * Bk * T2,
            "cols_mean": float(per.float().mean()), "cols_max": int(per.max()),
            "kept_cols_mean": float(perk.float().mean()), "kept_cols_max": int(perk.max()),
            "entries_per_region": float(tot / per.numel())}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
