"""Decompose the csr9 transfer time on C3: stream-only (all-zero kept bitmap:
no gathers / FMAs), full (all-ones bitmap), the real selection, and csr9.
Usage: python tools/csr9_decompose.py"""
import json
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
    import bench as B
    from paper_2203_12339_b200 import _lib
    from paper_2203_12339_b200.config import CONFIGS
    from paper_2203_12339_b200.runtime import csr9_layout

    _lib.load()
    cfg = CONFIGS["env_large_256"]
    g, b, dt, env, sc = B.setup_scene(cfg, 0, torch, {})
    sc.relight()
    n, K = sc.n, sc.K
    pcols, pvals, pieces, wbeg, W = csr9_layout(dt)
    xp = torch.empty((n, 4), dtype=torch.float64, device="cuda")
    bits = torch.empty((n + 31) // 32, dtype=torch.int32, device="cuda")
    sp = _lib.stream_ptr()
    _lib.call("sss_pack_x_bits", _lib.ptr(sc.x), n, _lib.ptr(xp), _lib.ptr(bits), sp)
    real = bits.clone()
    vk = torch.empty((K, 3, n), dtype=torch.float64, device="cuda")

    def run(bm):
        return lambda: _lib.call("sss_transfer_csr9s", K, n, _lib.ptr(pcols), _lib.ptr(pvals),
                                 _lib.ptr(pieces), _lib.ptr(wbeg), W, _lib.ptr(xp), _lib.ptr(bm),
                                 _lib.ptr(vk), sp)

    out = {}
    out["stream_only"] = timed(run(torch.zeros_like(bits)))
    out["all_ones"] = timed(run(torch.full_like(bits, -1)))
    out["real_selection"] = timed(run(real))
    out["csr9"] = timed(lambda: _lib.call("sss_transfer_csr9", K, n, _lib.ptr(pcols), _lib.ptr(pvals),
                                          _lib.ptr(pieces), _lib.ptr(wbeg), W, _lib.ptr(xp),
                                          _lib.ptr(vk), sp))
    sel = (sc.x != 0).any(dim=0)
    out["kept_col_frac"] = float(sel.float().mean())
    out["touched_frac"] = float(sel[dt.cols.long()].float().mean())
    out["padded_MB"] = pcols.numel() * 8 / 1e6
    out["stream_GBps"] = pcols.numel() * 8 / (out["stream_only"] * 1e-6) / 1e9
    print(json.dumps(out))


if __name__ == "__main__":
    main()
