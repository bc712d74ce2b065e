"""Upper bound of gather sharing inside flat16 warp iterations: per 512-entry
window (one warp iteration), the kept entries vs the distinct kept columns
(if every duplicate column sat in the same instruction slot, a window would
need one gather per distinct column). Usage: python tools/window_dup_stats.py"""
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
    sc.set_light(EnvLight(env.faces(11.0)))
    sc.relight()
    kept = (sc.x != 0).any(dim=0)
    n = dt.n
    kept_ext = torch.cat([kept, torch.zeros(1, dtype=torch.bool, device=kept.device)])
    out = {}
    for E in (16, 32):
        import os
        os.environ["SSS_FLAT16_E"] = str(E)
        sc.transfer_kernel = "flat16"
        dt.flat16 = None
        sc._launch_transfer(epilogue=False)
        torch.cuda.synchronize()
        pcols = dt.flat16[0].long() & 0xFFFFFFFF
        win = torch.arange(pcols.numel(), device=pcols.device) // (32 * E)
        m = kept_ext[pcols]
        key = win[m] * (n + 1) + pcols[m]
        uniq = torch.unique(key).numel()
        out[E] = {"kept_entries": int(m.sum()), "distinct_window_cols": uniq,
                  "max_gather_saving": 1 - uniq / max(1, int(m.sum()))}
        print(json.dumps({E: out[E]}), flush=True)


if __name__ == "__main__":
    main()
