"""Segment statistics of the C3 operator per (unit, band) item: how many
nonempty (row, k) segments an item has and how long they are — decides how
the transfer kernel should balance work. Usage: python tools/seg_stats.py"""
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
    n, K = dt.n, dt.K
    rp = dt.rowptr.cpu().numpy()
    cols = dt.cols.cpu().numpy().view(np.uint32).astype(np.int64)
    row_len = rp[:, 1:] - rp[:, :-1]
    out = {}
    for BW in (512, 1024, 2048, 4096):
        for rows_per_unit in (192, 256, 448):
            # per entry (k, row, band) -> segment counts
            k_of = np.repeat(np.arange(K), row_len.sum(axis=1))
            row_of = np.repeat(np.tile(np.arange(n), K), row_len.reshape(-1))
            band = cols // BW
            unit = row_of // rows_per_unit
            seg = (unit * (n // BW + 1) + band) * (K * rows_per_unit) + k_of * rows_per_unit + row_of % rows_per_unit
            segs, seg_len = np.unique(seg, return_counts=True)
            item = segs // (K * rows_per_unit)
            item_tot = np.bincount(item)
            item_nseg = np.bincount(item)
            nz = item_tot > 0
            seg_per_item = np.bincount(item)  # number of segments per item (ones weighted)
            ent_per_item = np.bincount(item, weights=seg_len)
            m = ent_per_item > 0
            out[f"BW{BW}_R{rows_per_unit}"] = {
                "items": int(m.sum()),
                "mean_entries_per_item": float(ent_per_item[m].mean()),
                "mean_segments_per_item": float(seg_per_item[m].mean()),
                "mean_entries_per_segment": float(seg_len.mean()),
                "p90_segment_len": float(np.percentile(seg_len, 90)),
                "max_segment_len": int(seg_len.max()),
            }
    print(json.dumps(out))


if __name__ == "__main__":
    main()
