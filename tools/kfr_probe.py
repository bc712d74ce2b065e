"""Where the kfr transfer's time goes on the C3 operator: the core launch
timed (CUDA events) with the frame's kept-column bitmap, with an all-clear
bitmap (no gathers, no value loads: stream + decode only) and an all-set
bitmap (every pair gathers and loads its values).

python tools/kfr_probe.py -> one JSON line
"""
import json
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def timed(f, reps=30):
    f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        f()
    e1.record()
    torch.cuda.synchronize()
    return 1e3 * e0.elapsed_time(e1) / reps


def main():
    import bench as B
    from paper_2203_12339_b200 import _lib
    from paper_2203_12339_b200.config import CONFIGS
    from paper_2203_12339_b200.runtime import EnvLight

    _lib.load()
    cfg = CONFIGS["env_large_256"]
    g, b, dt, env, sc = B.setup_scene(cfg, 0, torch, {})
    sc.set_light(EnvLight(env.faces(3.0)))
    bits = sc.xbits.clone()
    out = {"frame_bits_us": timed(sc.launch_transfer_core)}
    sc.xbits.zero_()
    out["no_kept_us"] = timed(sc.launch_transfer_core)
    sc.xbits.fill_(-1)
    sc.xbits[-1] = 0
    out["all_kept_us"] = timed(sc.launch_transfer_core)
    sc.xbits.copy_(bits)
    out["kept_fraction_of_cols"] = float((sc.x != 0).any(dim=0).float().mean())
    print(json.dumps(out))


if __name__ == "__main__":
    main()
