"""Pin the GPU precompute to the oracle at a BASELINE size (configs[1], C2:
128^2 geometry image, K = 8, 32 training materials, L = 3, step1_keep 5 %,
step2_fraction 0.95 — rule R1).

Run once in the build container (≈ 30-60 min of numpy on one core):

    python tests/golden/make_c2_digests.py

It writes
  * ``c2_inputs.npz``: the geometry image (f32 positions / normals / areas) and
    the PCA basis (r_nodes, bases, U, singular values, sigma nodes) — shipped as
    data so the GPU run sees the identical bits (numpy's SIMD transcendental
    and LAPACK paths may differ between hosts);
  * ``c2_digests.json``: per term k, SHA-256 of the oracle operator's cols
    (u32), colptr (i64), rowidx (u32) and f32-rounded vals, nnz, union size and
    kept / total energies.

``tests/test_gpu_precompute.py::test_c2_operator_matches_oracle_digests``
builds the operator on the GPU from c2_inputs.npz and compares. The oracle
(oracle/sss_oracle.py:precompute_compressed) is itself pinned bit for bit to
the real reference's precompute (tests/test_oracle_golden.py).
"""

from __future__ import annotations

import hashlib
import json
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, str(ROOT))


def digest(a, dtype):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=dtype).tobytes()).hexdigest()


def operator_digests(ops):
    out = []
    for op in ops:
        out.append({
            "nnz": int(op.rowidx.size), "n_cols": int(op.cols.size),
            "cols": digest(op.cols, "<u4"), "colptr": digest(op.colptr, "<i8"),
            "rowidx": digest(op.rowidx, "<u4"),
            "vals_f32": digest(np.asarray(op.vals).astype(np.float32), "<f4"),
            "kept_energy": float(op.kept_energy), "total_energy": float(op.total_energy),
            "step1_entries": int(op.step1_entries)})
    return out


def main():
    from oracle import sss_oracle as O
    from paper_2203_12339_b200 import config as C
    from paper_2203_12339_b200.basis import build_basis
    from paper_2203_12339_b200.geometry import make_geometry_image

    cfg = C.C2
    g = make_geometry_image(cfg.side, cfg.radius, cfg.bump_amp, cfg.bump_terms, cfg.seed)
    b = build_basis(cfg.K, cfg.lattice)
    np.savez_compressed(HERE / "c2_inputs.npz", side=cfg.side, positions=g.positions,
                        normals=g.normals, area=g.area, r_nodes=b.r_nodes, bases=b.bases,
                        singular_values=b.singular_values, sigma_nodes=b.sigma_nodes, U=b.U,
                        eta=b.eta, levels=cfg.levels, step1_keep=cfg.step1_keep,
                        step2_fraction=cfg.step2_fraction)
    t0 = time.time()
    ops = O.precompute_compressed(g.positions.astype(np.float64), g.area.astype(np.float64),
                                  cfg.side, b.r_nodes, b.bases, cfg.step1_keep,
                                  cfg.step2_fraction, levels=cfg.levels, w1="haar")
    secs = time.time() - t0
    out = {"config": cfg.name, "side": cfg.side, "K": cfg.K, "levels": cfg.levels,
           "step1_keep": cfg.step1_keep, "step2_fraction": cfg.step2_fraction,
           "oracle_seconds": round(secs, 1), "operators": operator_digests(ops)}
    (HERE / "c2_digests.json").write_text(json.dumps(out, indent=1) + "\n")
    print(json.dumps({"seconds": secs, "nnz": [o["nnz"] for o in out["operators"]]}))


if __name__ == "__main__":
    main()
