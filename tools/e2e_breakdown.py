"""Per-phase host timing of the public-API frame (Scene.set_light with a host
cubemap -> FrameResult) at C3: install (host->pinned->device), graph launch,
read-back enqueue, synchronize (GPU frame + copies), float64 arrays.
Usage: python tools/e2e_breakdown.py"""
import json
import sys
import time
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
    faces = [env.faces(float(f)) for f in range(60)]
    for f in range(5):
        sc.set_light(EnvLight(faces[f]))
    ph = {k: [] for k in ("install", "submit", "sync_and_result", "total")}
    for f in range(5, 55):
        t0 = time.perf_counter()
        sc._install_light(EnvLight(faces[f]))   # host staging (pinned), H2D deferred
        t1 = time.perf_counter()
        ev = sc._submit(sc._graph)              # sss_frame_replay: H2D, graph, widen, D2H
        t2 = time.perf_counter()
        fr = sc._frame({}, queued=True)         # synchronize + FrameResult arrays
        rad = fr.radiance
        t3 = time.perf_counter()
        for k, a_, b_ in (("install", t0, t1), ("submit", t1, t2), ("sync_and_result", t2, t3),
                          ("total", t0, t3)):
            ph[k].append((b_ - a_) * 1e3)
    out = {k: round(float(np.median(v)), 4) for k, v in ph.items()}
    out["gpu_graph_ms"] = round(ev[0].elapsed_time(ev[1]), 4)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
