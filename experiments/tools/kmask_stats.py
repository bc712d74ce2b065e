"""Padding cost of mask-sorted warp steps on the C3 operator: per row, pairs
sorted by k-mask (several orders), cut into 32-pair steps, each step storing
popc(OR of masks) x 32 values. Usage: python tools/kmask_stats.py"""
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
    k_of = np.repeat(np.arange(K), row_len.sum(axis=1))
    pair = row_of * n + cols
    up, inv = np.unique(pair, return_inverse=True)
    mask = np.zeros(up.size, np.int64)
    np.bitwise_or.at(mask, inv, 1 << k_of)
    prow = up // n
    pc = np.zeros(up.size, np.int64)
    for k in range(K):
        pc += (mask >> k) & 1
    out = {"pairs": int(up.size), "nnz": int(cols.size)}
    hist = np.bincount(mask, minlength=256)
    top = np.argsort(-hist)[:16]
    out["top_masks"] = [[int(m), int(hist[m])] for m in top]
    for name, key in (("mask", mask), ("popc_mask", pc * 256 + mask),
                      ("gray", mask ^ (mask >> 1))):
        o = np.lexsort((key, prow))
        m_s, r_s = mask[o], prow[o]
        # position within row
        rs = np.searchsorted(r_s, np.arange(n))
        pos = np.arange(up.size) - rs[r_s]
        step_id = r_s * 4096 + pos // 32
        us, sinv = np.unique(step_id, return_inverse=True)
        um = np.zeros(us.size, np.int64)
        np.bitwise_or.at(um, sinv, m_s)
        upc = np.zeros(us.size, np.int64)
        for k in range(K):
            upc += (um >> k) & 1
        stored = int((upc * 32).sum())
        out[name] = {"steps": int(us.size), "stored_vals": stored,
                     "pad_ratio": stored / cols.size,
                     "bytes": int(up.size * 4 + stored * 4 + us.size * 8)}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
