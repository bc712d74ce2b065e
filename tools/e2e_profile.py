"""Host-side profile of the public-API frame (Scene.set_light with a host
cubemap -> FrameResult): cProfile over 30 frames. Usage: python tools/e2e_profile.py"""
import cProfile
import io
import pstats
import sys
import time
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
    faces = [env.faces(float(f)) for f in range(40)]
    for f in range(5):
        sc.set_light(EnvLight(faces[f]))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for f in range(5, 35):
        sc.set_light(EnvLight(faces[f]))
    print("ms per frame", (time.perf_counter() - t0) / 30 * 1e3)
    pr = cProfile.Profile()
    pr.enable()
    for f in range(5, 35):
        sc.set_light(EnvLight(faces[f]))
    pr.disable()
    s = io.StringIO()
    pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(18)
    print(s.getvalue())


if __name__ == "__main__":
    main()
