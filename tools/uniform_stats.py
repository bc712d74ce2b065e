"""Lane utilisation of mask-uniform warp steps on the C3 operator: if every
step of a 32-row warp item processed ONE term mask (all lanes the same set of
terms, so the value decode and the FMAs are warp-uniform), how many lane
slots would be empty? Items = 32 consecutive tile-major rows of one term
group; per item and mask, steps = max over the 32 rows of their pair count
with that mask. Also the instruction estimate per item vs kfr's 94 per step.

python tools/uniform_stats.py -> one JSON line
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

    _lib.load()
    cfg = CONFIGS["env_large_256"]
    g, b, dt, env, sc = B.setup_scene(cfg, 0, torch, {})
    n, K = dt.n, dt.K
    row, k, col, _ = canonical_entries(dt)
    out = {}
    for G in (2, 4):
        NG = K // G
        key = (row * NG + k // G) * n + col
        u, inv = torch.unique(key, return_inverse=True)
        mask = torch.zeros(u.numel(), dtype=torch.int64, device=u.device).scatter_add_(
            0, inv, torch.bitwise_left_shift(torch.ones_like(k), k % G))
        rg = u // n                      # row * NG + group
        prow, pgrp = rg // NG, rg % NG
        nm = 1 << G
        cnt = torch.zeros((n, NG, nm), dtype=torch.int64, device=u.device)
        cnt.index_put_((prow, pgrp, mask), torch.ones_like(mask), accumulate=True)
        res = {}
        for rows_per_item in (32, 16):
            c = cnt.view(n // rows_per_item, rows_per_item, NG, nm)
            steps = c.amax(dim=1)               # (items, NG, nm)
            used = c.sum(dim=1)
            lanes = 32
            util = float(used.sum()) / float(lanes * steps.sum())
            pc = torch.tensor([bin(m).count("1") for m in range(nm)], device=u.device)
            # instructions: per step 6 + 5 * popc(mask)
            instr = float((steps * (6 + 5 * pc)).sum())
            res[f"rows_per_item_{rows_per_item}"] = {
                "lane_util": round(util, 4), "warp_steps": int(steps.sum()),
                "instr_estimate": instr}
        res["pairs"] = int(u.numel())
        out[f"G{G}"] = res
    out["kfr_reference"] = {"warp_steps": 1002356, "instr_per_step": 94, "instr": 94 * 1002356}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
