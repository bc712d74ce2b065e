"""Column-aligned sliced-ELL statistics of the C3 operator: for groups of G
receiver rows (tile-major, or re-ordered), the union of the group's columns
is the slot list; every slot holds one value per row (zero-padded). Per
frame only slots whose column is kept by some channel need their values
read. Reports the padding factor P = G * |union| / nnz and the per-frame
bytes of the kept slots (values G * 4 B, f32) for several groupings, per k
and K-fused (slot = column, values for all K terms of the G rows).

    python tools/ell_stats.py
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
    T2 = (1 << dt.levels) ** 2
    kept = []
    for f in range(4):
        sc.set_light(EnvLight(env.faces(f * 37.0)))
        kept.append((sc.x != 0).any(dim=0))
    rp = dt.rowptr.long()
    cols = dt.cols.long() & 0xFFFFFFFF
    nnz = int(rp[-1, -1])
    kk = torch.repeat_interleave(torch.arange(K, device="cuda"), rp[:, -1] - rp[:, 0])
    rows = torch.cat([torch.repeat_interleave(torch.arange(n, device="cuda"), torch.diff(rp[k]))
                      for k in range(K)])
    local = rows % T2
    tile = rows // T2
    # row orders: tile-major as stored; band-major (same local index across tiles)
    orders = {
        "tile_major": rows,
        "local_major": local * (n // T2) + tile,
    }
    out = {"nnz": nnz, "K": K, "frames": len(kept)}
    for G in (32, 64):
        for oname, rkey in orders.items():
            grp = rkey // G
            for fused in (False, True):
                gk = grp if fused else grp * K + kk
                key = gk * n + cols
                u = torch.unique(key)
                ucol = u % n
                slots = u.numel()
                vals_per_slot = G * (K if fused else 1)
                P = slots * vals_per_slot / nnz
                touched = [int(kf[ucol].sum()) for kf in kept]
                read = [t * vals_per_slot * 4 + slots * 2 for t in touched]
                out[f"G{G}/{oname}/{'kfused' if fused else 'perk'}"] = {
                    "slots": slots, "pad_factor": round(P, 3),
                    "kept_slot_frac": [round(t / slots, 3) for t in touched],
                    "read_MB_per_frame": [round(r / 1e6, 1) for r in read],
                }
                print(json.dumps({f"G{G}/{oname}/{fused}": out[f"G{G}/{oname}/{'kfused' if fused else 'perk'}"]}), flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
