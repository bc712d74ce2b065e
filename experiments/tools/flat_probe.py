"""Bandwidth probes on the C3 padded operator: plain read of the column and
value arrays, the flat-stream transfer without gathers (mode 1), with gathers
but no values (mode 2), and in full (mode 0). Usage: python tools/flat_probe.py"""
import ctypes as C
import json
import subprocess
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def timed(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, b in ev:
        a.record()
        fn()
        b.record()
    torch.cuda.synchronize()
    return float(np.median([a.elapsed_time(b) for a, b in ev])) * 1e3


def main():
    so = ROOT / "tools" / "_flat_probe.so"
    if True:
        subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17",
                               "-shared", "-Xcompiler", "-fPIC", "-o", str(so),
                               str(ROOT / "tools" / "flat_probe.cu")])
    P = C.CDLL(str(so))
    import bench as B
    from paper_2203_12339_b200 import _lib
    from paper_2203_12339_b200.config import CONFIGS
    from paper_2203_12339_b200.runtime import flat_layout

    _lib.load()
    cfg = CONFIGS["env_large_256"]
    g, b, dt, env, sc = B.setup_scene(cfg, 0, torch, {})
    sc.relight()
    n = sc.n
    out = {}
    for wps in (12, 16, 20):
        pcols, pvals, ne, heads, hpre, rowk, wbeg, W, st = flat_layout(dt, warps_per_sm=wps)
        xp = torch.empty((n, 4), dtype=torch.float64, device="cuda")
        bits = torch.empty((n + 31) // 32, dtype=torch.int32, device="cuda")
        _lib.call("sss_pack_x_bits", _lib.ptr(sc.x), n, _lib.ptr(xp), _lib.ptr(bits), _lib.stream_ptr())
        vk = torch.zeros((sc.K, 3, n), dtype=torch.float64, device="cuda")
        p = lambda t: C.c_void_p(t.data_ptr())
        for mode, ga in ((0, 1), (0, 2), (0, 3), (1, 2), (2, 1), (2, 2), (2, 3)):
            for skip in (False, True):
                bp = p(bits) if skip else None
                us = timed(lambda: P.probe_flat(mode, ga, n, p(pcols), p(pvals), C.c_uint(ne // 4),
                                                p(heads), p(hpre), p(rowk), p(wbeg), W, p(xp), bp,
                                                p(vk)))
                out[f"m{mode}_ga{ga}_w{wps}{'_skip' if skip else ''}"] = round(us, 1)
    acc = torch.zeros(1, dtype=torch.int64, device="cuda")
    for name, arr in (("cols", pcols), ("vals", pvals)):
        for grid in (148 * 8, 148 * 32):
            us = timed(lambda: P.probe_read(C.c_void_p(arr.data_ptr()), C.c_ulonglong(arr.numel() // 4),
                                            grid, C.c_void_p(acc.data_ptr())))
            out[f"read_{name}_g{grid}_GBps"] = arr.numel() * 4 / (us * 1e-6) / 1e9
    out["torch_sum_vals_GBps"] = pvals.numel() * 4 / (timed(lambda: pvals.sum()) * 1e-6) / 1e9
    out["entries"] = ne
    print(json.dumps(out))


if __name__ == "__main__":
    main()
