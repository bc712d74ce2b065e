"""K-fill of the C3 operator: for the union over k of (row, col) pairs, how
many of the K terms are present (fill = nnz / (pairs * K)). Usage:
python tools/kfill_stats.py"""
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
    row_of = np.repeat(np.tile(np.arange(n), K), row_len.reshape(-1))
    pair = row_of * n + cols
    up, cnt = np.unique(pair, return_counts=True)
    hist = np.bincount(cnt, minlength=K + 1)
    out = {"pairs": int(up.size), "nnz": int(cols.size), "fill": float(cols.size / (up.size * K)),
           "k_count_hist": hist.tolist(),
           "bytes_kfused_f32": int(up.size * (4 + 4 * K)),
           "bytes_csr": int(cols.size * 8)}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
