"""A/B of the transfer kernels on the C3 operator: per kernel, the core launch
timed alone with CUDA events (inputs prepared by a relight), v_k agreement
with kfr, and layout stats. Environment knobs (SSS_KFR_CHUNK, SSS_KFR_MINB)
apply to every Scene the tool builds.

    python tools/transfer_ab.py [kfr flat16]
"""
import json
import sys
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
    kerns = sys.argv[1:] or ["kfr", "flat16"]
    cfg = CONFIGS["env_large_256"]
    g, b, dt, env, sc = B.setup_scene(cfg, 0, torch, {})
    sc.set_light(EnvLight(env.faces(3.0)))
    ref = None
    out = {}
    for kern in ["kfr"] + [k for k in kerns if k != "kfr"]:
        sc.transfer_kernel = kern
        sc._graph = None
        sc.relight()
        sc.relight()
        vk = sc.vk.clone()
        if ref is None:
            ref = vk
        err = float((vk - ref).abs().max() / ref.abs().max())
        reps = 50
        sc.launch_transfer_core()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            sc.launch_transfer_core()
        e1.record()
        torch.cuda.synchronize()
        st = getattr(dt, kern, None)
        stats = st.stats if hasattr(st, "stats") else (st[-1] if isinstance(st, tuple) else None)
        if isinstance(stats, dict):  # the flat16 stats carry a device tensor (span_first)
            stats = {k: v for k, v in stats.items() if not torch.is_tensor(v)}
        out[kern] = {"us": 1e3 * e0.elapsed_time(e1) / reps, "rel_err_vs_kfr": err, "stats": stats}
        print(json.dumps({kern: out[kern]}), flush=True)


if __name__ == "__main__":
    main()
