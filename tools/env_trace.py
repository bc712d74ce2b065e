"""Phase timeline (us, CTA 0) of the environment projection kernel on the C3
cubemap. Usage: python tools/env_trace.py"""
import ctypes as C
import json
import subprocess
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]


def main():
    so = ROOT / "tools" / "_env_trace.so"
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17",
                           "-shared", "-Xcompiler", "-fPIC", "-o", str(so), str(ROOT / "tools" / "env_trace.cu")])
    P = C.CDLL(str(so))
    sys.path.insert(0, str(ROOT))
    from paper_2203_12339_b200 import lighting as LT

    env = LT.Environment(side=32, seed=7)
    faces = torch.as_tensor(env.faces(0.0), device="cuda")
    idx = torch.empty((3, 128), dtype=torch.int32, device="cuda")
    val = torch.empty((3, 128), dtype=torch.float64, device="cuda")
    out = (C.c_ulonglong * 16)()
    p = lambda t: C.c_void_p(t.data_ptr())
    for _ in range(3):
        P.env_trace(p(faces), 32, 128, p(idx), p(val), out)
    t = np.array(list(out), dtype=np.float64)
    names = ["start", "loaded", "haar", "radix", "applied", "compacted"]
    print(json.dumps({names[i]: round((t[i] - t[0]) / 1e3, 2) for i in range(6)}))


if __name__ == "__main__":
    main()
