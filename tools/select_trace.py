"""Phase timeline (us, CTA 0) of the cluster top-n select on the C3 spectrum.
Usage: python tools/select_trace.py"""
import ctypes as C
import json
import subprocess
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    so = ROOT / "tools" / "_select_trace.so"
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17",
                           "-shared", "-Xcompiler", "-fPIC", "-o", str(so),
                           str(ROOT / "tools" / "select_trace.cu")])
    P = C.CDLL(str(so))
    import bench as B
    from paper_2203_12339_b200 import _lib
    from paper_2203_12339_b200.config import CONFIGS

    _lib.load()
    g, b, dt, env, sc = B.setup_scene(CONFIGS["env_large_256"], 0, torch, {})
    sc.relight()
    keep = max(1, int(round(sc.e_keep * sc.n)))
    out = (C.c_ulonglong * 32)()
    p = lambda t: C.c_void_p(t.data_ptr())
    for _ in range(3):
        P.select_trace(p(sc.ehat), 3, sc.n, keep, p(sc.f2t), p(sc.x), p(sc.mask), p(sc.energy), out)
    t = np.array(list(out), dtype=np.float64)
    t0 = t[0]
    names = {0: "start", 1: "loaded"}
    for ps in range(8):
        names[2 + 3 * ps] = f"pass{ps}_hist"
        names[3 + 3 * ps] = f"pass{ps}_barrier"
        names[4 + 3 * ps] = f"pass{ps}_decided"
    names.update({26: "ties", 27: "applied", 28: "end"})
    print(json.dumps({names[i]: round((t[i] - t0) / 1e3, 2) for i in sorted(names) if t[i] > 0}))


if __name__ == "__main__":
    main()
