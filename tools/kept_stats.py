"""Structure of the kept-column set on C3 across several lights: kept
fraction and operator-entry share per tile-local Haar level class of the
column (tile-major column = tile * 4^L + local). Usage:
python tools/kept_stats.py"""
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
    from paper_2203_12339_b200.runtime import EnvLight

    _lib.load()
    cfg = CONFIGS["env_large_256"]
    g, b, dt, env, sc = B.setup_scene(cfg, 0, torch, {})
    n = dt.n
    T2 = (1 << dt.levels) ** 2
    local = torch.arange(n, device="cuda") % T2
    # class: 0 = DC, l = level (coarsest = 1 ... finest = L) of the local index
    lvl = torch.zeros(n, dtype=torch.long, device="cuda")
    for L in range(1, dt.levels + 1):
        lo = 4 ** (L - 1)
        hi = 4 ** L
        lvl[(local >= lo) & (local < hi)] = L
    col_nnz = torch.bincount(dt.cols.long(), minlength=n)
    out = {"levels": dt.levels, "classes": {}}
    kept_frames = []
    for f in range(6):
        sc.set_light(EnvLight(env.faces(f * 37.0)))
        kept_frames.append((sc.x != 0).any(dim=0))
    K = torch.stack(kept_frames).float()
    for L in range(dt.levels + 1):
        m = lvl == L
        out["classes"][str(L)] = {
            "cols": int(m.sum()),
            "kept_frac_per_frame": [round(float(K[i][m].mean()), 4) for i in range(K.shape[0])],
            "nnz_share": round(float(col_nnz[m].sum() / col_nnz.sum()), 4),
            "touched_share_of_nnz": [round(float((col_nnz[m] * K[i][m]).sum() / col_nnz.sum()), 4)
                                     for i in range(K.shape[0])],
        }
    out["touched_frac"] = [round(float((col_nnz * K[i]).sum() / col_nnz.sum()), 4) for i in range(K.shape[0])]
    # how stable is the kept set frame to frame
    out["jaccard_vs_frame0"] = [round(float((K[0] * K[i]).sum() / ((K[0] + K[i]) > 0).sum()), 4)
                                for i in range(K.shape[0])]
    print(json.dumps(out))


if __name__ == "__main__":
    main()
