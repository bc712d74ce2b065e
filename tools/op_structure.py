"""Structure of the C3 transfer operator as the frame sees it (design input
for the transfer kernel): entry shares by (row level class, column level
class), the share the current frame touches, row lengths, K-fill of
(row, column) pairs, column popularity, per-row-group distinct columns.
Usage: python tools/op_structure.py [config]  -> one JSON line."""
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
    cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "env_large_256"]
    g, b, dt, env, sc = B.setup_scene(cfg, 0, torch, {})
    n, K, L = dt.n, dt.K, dt.levels
    T2 = (1 << L) ** 2
    dev = "cuda"
    rp = dt.rowptr.to(dev)
    cols = dt.cols.to(dev).long() & 0xffffffff
    lens = (rp[:, 1:] - rp[:, :-1])  # (K, n)
    k_of = torch.repeat_interleave(torch.arange(K, device=dev), lens.sum(1))
    row_of = torch.repeat_interleave(torch.arange(n, device=dev).repeat(K), lens.reshape(-1))

    def cls(idx):
        loc = idx % T2
        c = torch.zeros_like(loc)
        for lv in range(1, L + 1):
            c[(loc >= 4 ** (lv - 1)) & (loc < 4 ** lv)] = lv
        return c

    rc, cc = cls(row_of), cls(cols)
    nnz = cols.numel()
    out = {"n": n, "K": K, "levels": L, "nnz": nnz, "nnz_per_k": [int(x) for x in dt.nnz_per_k]}
    tab = torch.zeros((L + 1, L + 1), dtype=torch.long, device=dev)
    tab.index_put_((rc, cc), torch.ones_like(rc), accumulate=True)
    out["share_row_x_col"] = (tab.double() / nnz).round(decimals=4).tolist()
    # frames
    kept = []
    for f in range(4):
        sc.set_light(EnvLight(env.faces(f * 25.0)))
        kept.append((sc.x != 0).cpu())
    kept_any = (kept[0] != 0).any(dim=0).to(dev)
    kept_c = kept[0].to(dev)  # (3, n)
    t_mask = kept_any[cols]
    ttab = torch.zeros_like(tab)
    ttab.index_put_((rc[t_mask], cc[t_mask]), torch.ones_like(rc[t_mask]), accumulate=True)
    touched = int(t_mask.sum())
    out["touched"] = touched
    out["touched_share_row_x_col"] = (ttab.double() / max(touched, 1)).round(decimals=4).tolist()
    out["touched_per_channel_entries"] = [int(kept_c[c][cols].sum()) for c in range(3)]
    cl_all = cls(torch.arange(n, device=dev))
    out["kept_frac_by_col_class"] = [[round(float(k[c][cl_all.cpu() == lv].float().mean()), 4)
                                      for lv in range(L + 1)] for k in kept[:1] for c in range(3)]
    out["kept_any_frac_by_col_class_frames"] = [
        [round(float((k != 0).any(0)[cl_all.cpu() == lv].float().mean()), 4) for lv in range(L + 1)]
        for k in kept]
    out["kept_any_frac"] = [round(float((k != 0).any(0).float().mean()), 4) for k in kept]
    # row lengths per (row, k), by row class
    rl = {}
    rcls = cls(torch.arange(n, device=dev))
    for lv in range(L + 1):
        m = rcls == lv
        x = lens[:, m].double()
        rl[str(lv)] = {"rows": int(m.sum()), "mean": round(float(x.mean()), 2),
                       "max": int(x.max()), "p50": float(x.median()),
                       "zero_frac": round(float((x == 0).double().mean()), 4)}
    out["row_len_by_row_class"] = rl
    # K-fill: distinct (row, col) pairs
    key = row_of * n + cols
    uk, cnt = torch.unique(key, return_counts=True)
    out["pairs"] = int(uk.numel())
    out["pair_k_fill_hist"] = torch.bincount(cnt, minlength=K + 1).tolist()
    tk = key[t_mask]
    out["touched_pairs"] = int(torch.unique(tk).numel())
    # column popularity
    cn = torch.bincount(cols, minlength=n)
    s, _ = torch.sort(cn, descending=True)
    cs = torch.cumsum(s, 0).double() / nnz
    out["top_cols_share"] = {str(t): round(float(cs[t - 1]), 4)
                             for t in (256, 1024, 2048, 4096, 8192, 16384, 32768)}
    tn = torch.bincount(cols[t_mask], minlength=n)
    s2, _ = torch.sort(tn, descending=True)
    cs2 = torch.cumsum(s2, 0).double() / max(touched, 1)
    out["top_touched_cols_share"] = {str(t): round(float(cs2[t - 1]), 4)
                                     for t in (256, 1024, 2048, 4096, 8192, 16384)}
    out["touched_distinct_cols"] = int((tn > 0).sum())
    # per row group: distinct touched columns (over its rows and all k)
    grp = {}
    for R in (64, 256, 1024, 4096):
        gk = (row_of[t_mask] // R) * n + cols[t_mask]
        ug = torch.unique(gk)
        per = torch.bincount(ug // n, minlength=n // R).double()
        ent = torch.bincount(row_of[t_mask] // R, minlength=n // R).double()
        grp[str(R)] = {"distinct_mean": round(float(per.mean()), 1), "distinct_max": int(per.max()),
                       "entries_mean": round(float(ent.mean()), 1),
                       "entries_per_distinct": round(float(ent.sum() / per.sum()), 2)}
    out["row_group_distinct_touched_cols"] = grp
    # by column class: entries per distinct column within 256-row groups
    # tile-of-col locality: |tile(row) - tile(col)| in tile units (2D)
    ts = (1 << 0)  # noqa
    tiles_side = dt.side >> L
    tr, tcol = row_of // T2, cols // T2
    dy = (tr // tiles_side - tcol // tiles_side).abs()
    dx = (tr % tiles_side - tcol % tiles_side).abs()
    d = torch.maximum(dx, dy)
    out["tile_cheb_dist_hist_touched"] = torch.bincount(
        torch.clamp(d[t_mask], max=33), minlength=34).tolist()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
