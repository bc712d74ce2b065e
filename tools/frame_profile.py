"""Per-kernel device times of one C3 frame (CUDA events around each launch,
repeated, warm) — a quick breakdown next to the ncu launch list.

    python tools/frame_profile.py [--side 256] [--reps 20]
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


def timed(fn, reps):
    s = torch.cuda.current_stream()
    fn()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, b in ev:
        a.record(s)
        fn()
        b.record(s)
    torch.cuda.synchronize()
    return float(np.median([a.elapsed_time(b) for a, b in ev])) * 1e3  # us


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--side", type=int, default=256)
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    import bench as B
    from paper_2203_12339_b200 import _lib
    from paper_2203_12339_b200.config import CONFIGS

    cfg = CONFIGS["env_large_256"].with_(side=a.side)
    _lib.load()
    stats = {}
    g, b, dt, env, sc = B.setup_scene(cfg, 0, torch, stats)
    sc.relight()
    sp = _lib.stream_ptr()
    s, kk = sc._light_kind[1], sc.env_keep
    out = {}
    out["env_project+union"] = timed(lambda: _lib.call(
        "sss_env_project", _lib.ptr(sc.light_buf), s, kk, _lib.ptr(sc.env_idx), _lib.ptr(sc.env_val),
        _lib.ptr(sc.env_uidx), _lib.ptr(sc.env_ulc), _lib.ptr(sc.env_nu), sp), a.reps)
    out["env_irradiance_sel+haar"] = timed(lambda: _lib.call(
        "sss_env_irradiance_sel", _lib.ptr(sc.W2), 6 * s * s, _lib.ptr(sc.env_idx),
        _lib.ptr(sc.env_val), kk, sc.side, sc.levels, None, _lib.ptr(sc.ehat), sp), a.reps)
    out["env_irradiance+haar"] = timed(lambda: _lib.call(
        "sss_env_irradiance", _lib.ptr(sc.W2), 6 * s * s, _lib.ptr(sc.env_uidx), _lib.ptr(sc.env_ulc),
        _lib.ptr(sc.env_nu), kk, sc.side, sc.levels, None, _lib.ptr(sc.ehat), sp), a.reps)
    keep = max(1, int(round(sc.e_keep * sc.n)))
    out["select_topn"] = timed(lambda: _lib.call(
        "sss_select_topn", _lib.ptr(sc.ehat), 3, sc.n, keep, _lib.ptr(sc.f2t), _lib.ptr(sc.x),
        _lib.ptr(sc.mask), _lib.ptr(sc.energy), sp), a.reps)
    out["material_weights"] = timed(sc._launch_weights, a.reps)
    ref_vk = None
    for kern in ("kfr", "flat16"):
        sc.transfer_kernel = kern
        sc.vk.fill_(float("nan"))
        sc._launch_transfer()
        torch.cuda.synchronize()
        out[f"finite_{kern}"] = bool(torch.isfinite(sc.vk).all())
        out[f"transfer_{kern}"] = timed(sc._launch_transfer, a.reps)
        if ref_vk is None:
            ref_vk = sc.vk.clone()
        else:
            out[f"relerr_{kern}"] = float((sc.vk - ref_vk).abs().max() / ref_vk.abs().max())
    out.update({f"kfr_{k}": v for k, v in dt.kfr.stats.items()})
    sc.transfer_kernel = "kfr"
    out["edit_finish"] = timed(sc._launch_edit, a.reps)
    sc.capture()
    out["relight_graph"] = timed(lambda: sc.replay(False), a.reps)
    out["edit_graph"] = timed(lambda: sc.replay(True), a.reps)
    out["operator_nnz"] = dt.nnz
    out["operator_MB"] = dt.nnz * 8 / 1e6
    print(json.dumps({k: (v if k.startswith("relerr") else round(v, 2)) if isinstance(v, float) else v
                      for k, v in out.items()}))


if __name__ == "__main__":
    main()
