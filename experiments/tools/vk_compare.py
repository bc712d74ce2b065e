"""Sanity probe for the kernel A/B comparisons: v_k of two transfer kernels on
the C3 frame, max abs difference, number of differing elements, and the
magnitudes involved. Usage: python tools/vk_compare.py kernA kernB"""
import json
import os
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import bench as B
    from paper_2203_12339_b200 import _lib
    from paper_2203_12339_b200.config import CONFIGS

    ka, kb = sys.argv[1], sys.argv[2]
    _lib.load()
    g, b, dt, env, sc = B.setup_scene(CONFIGS["env_large_256"], 0, torch, {})
    sc.relight()
    sc.transfer_kernel = ka
    sc.vk.fill_(float("nan"))
    sc._launch_transfer()
    torch.cuda.synchronize()
    va = sc.vk.clone()
    os.environ["SSS_X_F32"] = os.environ.get("SSS_X_F32_B", "0")
    sc.transfer_kernel = kb
    sc.vk.fill_(float("nan"))
    sc._launch_transfer()
    torch.cuda.synchronize()
    vb = sc.vk.clone()
    d = (va - vb).abs()
    out = {"a": ka, "b": kb, "max_abs_diff": float(d.max()), "n_diff": int((d > 0).sum()),
           "n": d.numel(), "max_abs": float(va.abs().max()), "n_nonzero": int((va != 0).sum()),
           "x_nonzero_cols": int((sc.x != 0).any(dim=0).sum()),
           "sample_a": va.view(-1)[:4].tolist(), "sample_b": vb.view(-1)[:4].tolist()}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
