"""Row-block CSC statistics of the C3 operator (design probe for the
row-block column-major transfer): for row blocks of RB tile-major rows, the
number of (block, column) segments over all K terms, the segments whose
column is kept in a frame, the entries they hold, and per-block balance.

    python tools/csc_block_stats.py
"""
import json
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import bench as B
    from paper_2203_12339_b200 import _lib
    from paper_2203_12339_b200.config import CONFIGS
    from paper_2203_12339_b200.runtime import EnvLight

    _lib.load()
    cfg = CONFIGS["env_large_256"]
    g, b, dt, env, sc = B.setup_scene(cfg, 0, torch, {})
    n, K = dt.n, dt.K
    sc.set_light(EnvLight(env.faces(11.0)))
    kept = (sc.x != 0).any(dim=0)
    rp = dt.rowptr.long()
    cols = dt.cols.long() & 0xFFFFFFFF
    rows = torch.cat([torch.repeat_interleave(torch.arange(n, device="cuda"), torch.diff(rp[k]))
                      for k in range(K)])
    out = {}
    for RB in (128, 256, 512, 1024):
        key = (rows // RB) * n + cols
        u, cnt = torch.unique(key, return_counts=True)
        kc = kept[u % n]
        per_block = torch.bincount(u // n, weights=cnt.double(), minlength=n // RB)
        kept_per_block = torch.bincount(u // n, weights=(cnt * kc).double(), minlength=n // RB)
        out[RB] = {"segments": int(u.numel()), "kept_segments": int(kc.sum()),
                   "kept_entries": int(cnt[kc].sum()),
                   "mean_seg_len": float(cnt.double().mean()),
                   "kept_entries_per_block_max_over_mean":
                       float(kept_per_block.max() / kept_per_block.mean()),
                   "entries_per_block_max_over_mean": float(per_block.max() / per_block.mean())}
        print(json.dumps({RB: out[RB]}), flush=True)


if __name__ == "__main__":
    main()
