"""How much of the C3 operator a frame must read when unkept columns are
skipped at a given granularity (the design input of the column-skipping
transfer). For several frames of the bench sequence: x's kept columns
(any channel), and for groups keyed by (receiver row block, column group)
the share of stored entries lying in groups with >= 1 kept column.

python tools/block_skip_stats.py  ->  one JSON line
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
    from paper_2203_12339_b200.layout import canonical_entries
    from paper_2203_12339_b200.runtime import EnvLight

    _lib.load()
    cfg = CONFIGS["env_large_256"]
    g, b, dt, env, sc = B.setup_scene(cfg, 0, torch, {})
    n, L = dt.n, dt.levels
    T2 = 4 ** L
    row, k, col, val = canonical_entries(dt)
    del val
    nnz = row.numel()
    loc = col % T2
    lvl = torch.zeros_like(loc)
    for l in range(1, L + 1):
        lvl[(loc >= 4 ** (l - 1)) & (loc < 4 ** l)] = l
    out = {"nnz": nnz, "n": n, "levels": L, "frames": []}
    out["nnz_share_by_level"] = [round(float((lvl == l).sum()) / nnz, 4) for l in range(L + 1)]
    # distinct (row, col) pairs and per-level pair share
    pair = row * n + col
    up = torch.unique(pair)
    out["pairs"] = int(up.numel())
    kept_frames = []
    for f in range(0, 60, 12):
        sc.set_light(EnvLight(env.faces(f * 1.0)))
        kept_frames.append((sc.x != 0).any(dim=0))
    for kept in kept_frames:
        fr = {}
        kc = kept[col]
        fr["touched"] = round(float(kc.sum()) / nnz, 4)
        fr["touched_by_level"] = [round(float((kc & (lvl == l)).sum()) / max(int((lvl == l).sum()), 1), 4)
                                  for l in range(L + 1)]
        fr["kept_cols_by_level"] = []
        cl = torch.arange(n, device=kept.device) % T2
        clv = torch.zeros_like(cl)
        for l in range(1, L + 1):
            clv[(cl >= 4 ** (l - 1)) & (cl < 4 ** l)] = l
        for l in range(L + 1):
            fr["kept_cols_by_level"].append(round(float(kept[clv == l].float().mean()), 4))
        # skip granularity: column groups of the fine level(s) by source tile
        tile = col // T2
        for name, gkey_col in [("src_tile", torch.arange(n, device=kept.device) // T2),
                               ("src_tile_level", (torch.arange(n, device=kept.device) // T2) * 8 + clv),
                               ("col8", torch.arange(n, device=kept.device) // 8),
                               ("col4", torch.arange(n, device=kept.device) // 4)]:
            ng = int(gkey_col.max()) + 1
            gk = torch.zeros(ng, dtype=torch.bool, device=kept.device)
            gk.index_put_((gkey_col,), kept, accumulate=True)
            need = gk[gkey_col[col]]
            fr[f"read_share_{name}"] = round(float(need.sum()) / nnz, 4)
            fine = lvl == L
            fr[f"read_share_{name}_fine"] = round(float((need & fine).sum()) / max(int(fine.sum()), 1), 4)
        out["frames"].append(fr)
        del kc
    # entries per (receiver tile, source tile) block and per (row block 32, source tile)
    rt = row // T2
    blk = rt * (n // T2) + tile
    cnt = torch.bincount(blk)
    nzb = cnt[cnt > 0]
    out["rtile_stile_blocks"] = int(nzb.numel())
    out["entries_per_block_mean"] = round(float(nzb.float().mean()), 2)
    out["entries_per_block_q"] = [int(x) for x in torch.quantile(nzb.float(), torch.tensor(
        [0.1, 0.5, 0.9], device=nzb.device)).tolist()]
    # distinct columns per 64-row receiver tile (all k), fine only
    fine = lvl == L
    key = rt[fine] * n + col[fine]
    uk = torch.unique(key)
    out["fine_cols_per_rtile_mean"] = round(float(uk.numel()) / (n // T2), 1)
    out["fine_entries_per_rtile_mean"] = round(float(fine.sum()) / (n // T2), 1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
