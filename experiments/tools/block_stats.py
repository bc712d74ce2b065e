"""Block-sparse fill of the C3 operator in tile-major (row, column) space: for
block shapes (rb x cb), nonzero blocks and fill = nnz / (blocks * rb * cb).
Usage: python tools/block_stats.py"""
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
    k_of = np.repeat(np.arange(K), row_len.sum(axis=1))
    row_of = np.repeat(np.tile(np.arange(n), K), row_len.reshape(-1))
    out = {}
    for rb, cb in ((2, 4), (4, 4), (4, 8), (8, 4), (8, 8), (2, 8), (16, 4), (4, 16), (8, 16), (16, 8)):
        key = (k_of * (n // rb) + row_of // rb) * (n // cb) + cols // cb
        nb = np.unique(key).size
        out[f"{rb}x{cb}"] = {"blocks": int(nb), "fill": float(cols.size / (nb * rb * cb)),
                             "x_loads_per_nnz": float(nb * cb / cols.size)}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
