"""Load-balance statistics of the v5 stream layout (per item: max / mean
entries per consumer thread and per warp). Usage: python tools/v4_balance.py"""
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
    from paper_2203_12339_b200.stream4 import HDR, NW, TPU, build_v4

    _lib.load()
    cfg = CONFIGS["env_large_256"]
    stats = {}
    g, b, dt, env, sc = B.setup_scene(cfg, 0, torch, stats)
    lay = build_v4(dt)
    items = lay.items.cpu().numpy().view(np.dtype([("off", "<u8"), ("bytes", "<u4"),
                                                   ("band", "<u2"), ("pad", "<u2")]))
    stream = lay.stream.cpu().numpy()
    nit = len(items)
    counts = np.stack([stream[o + 2 * (NW + 1): o + 2 * (NW + 1) + 2 * TPU].view("<u2")
                       for o in items["off"]]).astype(np.int64)
    per_warp_max = counts.reshape(nit, NW, 32).max(axis=2)
    out = {
        "items": nit,
        "mean_entries_per_thread": float(counts.mean()),
        "mean_max_thread": float(counts.max(axis=1).mean()),
        "mean_max_warp_lane": float(per_warp_max.mean()),
        "critical_over_mean": float(counts.max(axis=1).sum() / counts.mean(axis=1).sum()),
        "unit_total_spread": None,
    }
    u_item0 = lay.unit_item0.cpu().numpy()
    u_n = lay.unit_nitems.cpu().numpy()
    tot = [counts[a:a + n].sum() for a, n in zip(u_item0, u_n)]
    crit = [counts[a:a + n].max(axis=1).sum() for a, n in zip(u_item0, u_n)]
    thread_tot = [counts[a:a + n].sum(axis=0) for a, n in zip(u_item0, u_n)]
    out["unit_entries_min_max"] = [int(min(tot)), int(max(tot))]
    out["unit_critical_path_max"] = int(max(crit))
    out["thread_total_max_over_mean"] = float(np.mean([t.max() / t.mean() for t in thread_tot]))
    print(json.dumps(out))


if __name__ == "__main__":
    main()
