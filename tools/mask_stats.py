"""Term-mask structure of the C3 operator's (row, term group, column) pairs
for term groups of G = 1, 2, 4, 8: pair counts, mean terms per pair, kept
(touched) pairs of a bench frame, the commonest masks, and the kfr layout's
own stream statistics. Design input of the transfer kernel.

python tools/mask_stats.py  ->  one JSON line
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
    from paper_2203_12339_b200.layout import canonical_entries, kfr_layout
    from paper_2203_12339_b200.runtime import EnvLight

    _lib.load()
    cfg = CONFIGS["env_large_256"]
    g, b, dt, env, sc = B.setup_scene(cfg, 0, torch, {})
    sc.set_light(EnvLight(env.faces(3.0)))
    kept = (sc.x != 0).any(dim=0)
    n, K = dt.n, dt.K
    row, k, col, _ = canonical_entries(dt)
    out = {"nnz": row.numel(), "K": K}
    T2 = 4 ** dt.levels
    loc = col % T2
    fine = loc >= 4 ** (dt.levels - 1)
    for G in (1, 2, 4, 8):
        NG = (K + G - 1) // G
        key = ((row * NG + k // G) * n + col)
        u, inv = torch.unique(key, return_inverse=True)
        mask = torch.zeros(u.numel(), dtype=torch.int64, device=u.device).scatter_add_(
            0, inv, torch.bitwise_left_shift(torch.ones_like(k), k % G))
        pc = torch.zeros(u.numel(), dtype=torch.int64, device=u.device).scatter_add_(
            0, inv, torch.ones_like(k))
        pcol = u % n
        pk = kept[pcol]
        d = {"pairs": int(u.numel()), "terms_per_pair": round(float(pc.float().mean()), 3),
             "kept_pairs": int(pk.sum()), "kept_terms_per_pair": round(float(pc[pk].float().mean()), 3)}
        if G >= 4:
            grp = (u // n) % NG
            for gi in range(NG):
                m = mask[grp == gi]
                h = torch.bincount(m, minlength=1 << G)
                top = torch.argsort(h, descending=True)[:8]
                d[f"g{gi}_top_masks"] = {format(int(t), f"0{G}b")[::-1]: round(float(h[t]) / m.numel(), 3)
                                         for t in top}
        out[f"G{G}"] = d
    # per term: entries and fine share
    out["entries_per_k"] = [int((k == i).sum()) for i in range(K)]
    out["fine_share_per_k"] = [round(float((fine & (k == i)).sum()) / max(int((k == i).sum()), 1), 3)
                               for i in range(K)]
    lay = kfr_layout(dt)
    out["kfr_stats"] = lay.stats
    out["kfr_stream_bytes"] = int(lay.stream.numel() * 4)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
