"""Kernel timeline of the captured C3 relight graph (CUPTI via torch.profiler):
per kernel, start offset inside the frame and duration, medians over the
replays - shows the gaps between dependent kernels that per-kernel timings
and ncu's serialized launch list cannot.

    python tools/graph_timeline.py [--reps 10]
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    import bench as B
    from paper_2203_12339_b200 import _lib
    from paper_2203_12339_b200.config import CONFIGS
    from torch.profiler import ProfilerActivity, profile

    cfg = CONFIGS["env_large_256"]
    _lib.load()
    g, b, dt, env, sc = B.setup_scene(cfg, 0, torch, {})
    for _ in range(3):
        sc.relight()
    if sc._graph is None:
        sc.capture()
    for _ in range(5):
        sc.replay()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        for _ in range(a.reps):
            sc.replay()
            torch.cuda.synchronize()
    evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    evs.sort(key=lambda e: e.time_range.start)
    # split into frames at k_env_project (first kernel of the chain)
    frames, cur = [], []
    for e in evs:
        if "env_project" in e.name and cur:
            frames.append(cur)
            cur = []
        cur.append(e)
    if cur:
        frames.append(cur)
    frames = [f for f in frames if any("transfer" in e.name for e in f)]
    rows = {}
    for f in frames:
        t0 = min(e.time_range.start for e in f)
        for e in f:
            name = e.name.split("(")[0].replace("void ", "").replace("sss::", "")[:40]
            rows.setdefault(name, []).append((e.time_range.start - t0, e.time_range.end - t0))
    out = []
    for name, v in rows.items():
        s = float(np.median([x[0] for x in v]))
        t = float(np.median([x[1] for x in v]))
        out.append({"kernel": name, "start_us": round(s, 2), "end_us": round(t, 2), "dur_us": round(t - s, 2)})
    out.sort(key=lambda r: r["start_us"])
    res = {"frames": len(frames), "timeline": out,
           "frame_span_us": round(max(r["end_us"] for r in out), 2)}
    print(json.dumps(res, indent=1))
    if a.out:
        Path(a.out).write_text(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
