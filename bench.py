"""Headline benchmark: the 256x256 environment-lit relight + material-edit
frame (BASELINE.json configs[2], "C3") on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A step is one frame of the C3 sequence: the cubemap rotates 1 deg about +y
(relight: env projection -> E -> w0 Haar -> top-n -> K-fused transfer +
recombine + inverse Haar + shade), and every 10th frame also applies a
material edit (edit path). ``value`` = shaded points/s with inputs resident
in HBM (CUDA graphs, device timing); ``e2e`` = the same through the public
Scene API with host cubemaps in and host radiance out. Under torchrun every
rank renders its own independent object (weak scaling, no data-path
collective); timing is the max over ranks.

``--impl reference`` times the reference's own implementation of the same
frames on the host cores (rank 0 only): whole frames of the same sequence
through sssrelight from baseline/_ref (oracle/reference_frame.py), on an
operator exported by a separate GPU process as a PRTS1 file and loaded with
the reference's own loader (the timing process never maps this framework's
library).
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "shaded points/sec & ms per relight+material-edit frame; % of HBM roofline"
UNIT = "shaded points/s"


def _args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="env_large_256")
    ap.add_argument("--cpu-frames", type=int, default=3,
                    help="frames of the reference path timed for cpu_baseline")
    ap.add_argument("--export-operator", default=None,
                    help=argparse.SUPPRESS)  # internal: the reference arm's GPU export step
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--side", type=int, default=None, help="override the geometry-image side (testing)")
    ap.add_argument("--no-secondary", action="store_true",
                    help="skip the C4 sweep / C5 pair-pass measurements in the JSON line")
    return ap.parse_args()


def _peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md)."""

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = Path("/tmp") / f"sss_clocks_{os.getpid()}.csv"

    def start(self):
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm,"
                 "clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap", "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=self.fh, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
            return
        # nvidia-smi's start-up (NVML init) stalls GPU work submission for
        # milliseconds: let it finish (first sample written) before the timed
        # region, which the 100 ms samples then span
        t0 = time.time()
        while time.time() - t0 < 3.0 and self.proc.poll() is None:
            if self.path.stat().st_size > 0:
                break
            time.sleep(0.005)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        self.proc.wait()
        self.fh.close()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.path.read_text().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for nm, v in zip(names, f[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(mx)), "reasons": sorted(reasons),
                "samples": len(sm)}


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def max_over_ranks(x: float, ws: int, device="cuda") -> float:
    """The job's time is the slowest rank's (timing rule: max over ranks)."""
    if ws <= 1:
        return float(x)
    import torch

    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    return float(t.item())


def whole_job_rate(points_per_rank: int, ws: int, steps: int, ms: float) -> float:
    """Weak scaling: every rank renders its own object of `points_per_rank`
    points per step; the job's rate is all ranks' points over the slowest
    rank's time."""
    return ws * points_per_rank * steps / (ms / 1e3)


def workload_config(cfg, n, nnz, ws):
    """The `config` object of the JSON line: identical for both arms."""
    return {
        "workload": f"{cfg.name} (BASELINE configs[2], C3): relight per frame, edit every "
                    f"{cfg.extra.get('edit_every', 10)}",
        "side": cfg.side, "points": n, "K": cfg.K, "training_materials": cfg.n_materials,
        "levels": cfg.levels, "step1_keep": cfg.step1_keep, "step2_fraction": cfg.step2_fraction,
        "e_keep": cfg.e_keep,
        "env": f"6x{cfg.env_side}x{cfg.env_side} cubemap, top-128 per channel, "
               f"{cfg.extra.get('rotate_deg', 1.0)} deg/frame about +y",
        "operator_nnz": int(nnz),
        "l2": "inputs larger than L2 (operator > 0.5 GB vs 126 MB L2)",
        "parallelism": f"{ws} independent objects (1 per GPU)" if ws > 1 else "1 GPU",
    }


def setup_scene(cfg, rank, torch, stats):
    from paper_2203_12339_b200 import lighting as LT
    from paper_2203_12339_b200.basis import OpticalMaterial, build_basis
    from paper_2203_12339_b200.geometry import make_geometry_image
    from paper_2203_12339_b200.precompute import precompute_compressed
    from paper_2203_12339_b200.runtime import EnvLight, Scene

    g = make_geometry_image(cfg.side, cfg.radius, cfg.bump_amp, cfg.bump_terms, cfg.seed + rank)
    b = build_basis(cfg.K, cfg.lattice)
    t0 = time.perf_counter()
    dt = precompute_compressed(g, b, cfg.levels, cfg.step1_keep, cfg.step2_fraction, stats=stats)
    torch.cuda.synchronize()
    stats["precompute_s"] = time.perf_counter() - t0
    env = LT.Environment(side=cfg.env_side, seed=7 + rank)
    m0 = OpticalMaterial(sigma_s_prime=cfg.material[0], sigma_a=cfg.material[1], eta=cfg.material[2])
    scene = Scene(g, dt, b, m0, EnvLight(env.faces(0.0)), e_keep=cfg.e_keep)
    return g, b, dt, env, scene


def frame_inputs(cfg, env, n_frames, seed):
    """Host inputs of the C3 sequence: rotated cubemaps and edit materials."""
    from paper_2203_12339_b200.basis import OpticalMaterial
    from paper_2203_12339_b200.config import SIGMA_BOX

    rng = np.random.default_rng(seed)
    faces = [env.faces(cfg.extra.get("rotate_deg", 1.0) * f) for f in range(n_frames)]
    mats = {}
    every = cfg.extra.get("edit_every", 10)
    for f in range(n_frames):
        if f % every == every - 1:
            sp = np.exp(rng.uniform(np.log(SIGMA_BOX[0]), np.log(SIGMA_BOX[1]), 3))
            sa = np.exp(rng.uniform(np.log(SIGMA_BOX[2]), np.log(SIGMA_BOX[3]), 3))
            mats[f] = OpticalMaterial(sigma_s_prime=sp, sigma_a=sa, eta=cfg.material[2])
    return faces, mats


def run_ours(a, cfg):
    import torch

    ws, rank, local = _dist()
    torch.cuda.set_device(local)
    if ws > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl")
    from paper_2203_12339_b200 import _lib

    _lib.load()
    stats = {}
    g, b, dt, env, scene = setup_scene(cfg, rank, torch, stats)
    n = g.count
    total = a.warmup + a.steps
    faces, mats = frame_inputs(cfg, env, total, 100 + rank)
    dev_faces = torch.stack([torch.as_tensor(f) for f in faces]).cuda()
    dev_mats = {f: torch.tensor(np.concatenate([m.sigma_s_prime, m.sigma_a, [m.eta]]),
                                dtype=torch.float64).cuda() for f, m in mats.items()}
    scene.capture()
    stream = torch.cuda.current_stream()

    def step(f):
        scene.light_buf.copy_(dev_faces[f], non_blocking=True)
        scene.replay(edit=False)
        if f in dev_mats:
            scene.material_buf.copy_(dev_mats[f], non_blocking=True)
            scene.replay(edit=True)

    for f in range(a.warmup):
        step(f)
    torch.cuda.synchronize()
    if ws > 1:
        torch.distributed.barrier()
    clocks = Clocks(local)
    clocks.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_push("timed")  # ncu --nvtx-include "timed/" launch lists
    e0.record(stream)
    for f in range(a.warmup, total):
        step(f)
    e1.record(stream)
    torch.cuda.nvtx.range_pop()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    clk = clocks.stop()
    ms = max_over_ranks(ms, ws)
    n_edit = sum(1 for f in range(a.warmup, total) if f in dev_mats)
    ms_per_step = ms / a.steps
    value = whole_job_rate(n, ws, a.steps, ms)

    # ---- dominant kernel: the K-fused transfer, timed alone on its stream
    kt = []
    for f in range(min(a.steps, 20)):
        ka, kb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ka.record(stream)
        scene.launch_transfer_core()
        kb.record(stream)
        kt.append((ka, kb))
    torch.cuda.synchronize()
    k_ms = float(np.mean([x.elapsed_time(y) for x, y in kt]))
    kname = scene.transfer_kernel
    kchoice = dict(scene.transfer_timings_us)
    # algorithmic bytes of one transfer launch (SURVEY §8d B_T + B_c), with the
    # selection of the current frame: entries whose w0 column is kept by any
    # channel (8 B each: u32 col + f32 val) + row pointers + v_k cache write +
    # radiance writes + geometry reads
    sel = (scene.x != 0).any(dim=0)
    touched = int(sel[dt.cols.long()].sum().item())
    n_kept = int(sel.sum().item())
    K = dt.K
    # algorithmic bytes of the timed launch (SURVEY §8d B_T): 8 B per touched
    # coefficient (u32 column + f32 value, the reference container's width),
    # 8 B per selected column and term (+1), and the v_k write (K x 3 x N fp64,
    # the stage-2 cache). The kernel's own packing of x / the kept bitmap and
    # the radiance / geometry of the edit epilogue are not part of this launch
    alg_bytes = 8 * touched + 8 * K * (n_kept + 1) + 24 * K * n
    all_bytes = 8 * dt.nnz + 8 * K * (n + 1) + 24 * K * n
    peak, peak_kind = _peaks()
    achieved = alg_bytes / (k_ms / 1e3) / 1e9
    traffic_path = ROOT / "profiles" / f"r02_transfer_{scene.transfer_kernel}_dram_bytes.json"
    traffic = None
    if traffic_path.exists():
        try:
            traffic = json.loads(traffic_path.read_text()).get("dram_bytes_per_launch")
        except Exception:
            traffic = None

    # ---- e2e: public API, host cubemap in, host radiance out
    from paper_2203_12339_b200.runtime import EnvLight

    n_e2e = min(a.steps, 100)
    # untimed API frames first: allocate the pinned read-back blocks and warm
    # the host path (as the W warm-up steps do for the device loop)
    for f in range(min(a.warmup, 5) or 1):  # the read-back block pool reaches steady state
        fr = scene.set_light(EnvLight(faces[f]))
        fr = scene.set_material(scene.material)
    del fr
    torch.cuda.synchronize()
    if ws > 1:
        torch.distributed.barrier()
    # three blocks of the same n_e2e-frame sequence; the median block (the
    # host shares the box: single blocks occasionally stall by 30-50 %)
    blocks = []
    for _blk in range(3):
        t0 = time.perf_counter()
        for i in range(n_e2e):
            f = a.warmup + i
            fr = scene.set_light(EnvLight(faces[f]))
            if f in mats:
                fr = scene.set_material(mats[f])
        torch.cuda.synchronize()
        blocks.append(time.perf_counter() - t0)
    e2e_s = float(np.median(blocks))
    e2e_s = max_over_ranks(e2e_s, ws)
    n_edit_e2e = sum(1 for i in range(n_e2e) if a.warmup + i in mats)
    h2d = faces[0].nbytes + (56 * n_edit_e2e) / n_e2e
    d2h = (2 * n * 3 * 8 + 48) * (1 + n_edit_e2e / n_e2e)  # f64 radiance + unclamped + energies
    e2e = {"value": ws * n * n_e2e / e2e_s, "unit": UNIT, "ms_per_step": 1e3 * e2e_s / n_e2e,
           "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h), "steps": n_e2e,
           "timing": "median of 3 blocks of the sequence (wall clock, synchronize at block end)",
           "block_ms_per_step": [round(1e3 * b_ / n_e2e, 4) for b_ in blocks],
           "path": "Scene.set_light(EnvLight(host cubemap)) / set_material -> FrameResult (numpy)"}

    # ---- edit-path latency alone (launch-bound; reported separately)
    ee = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ee[0].record(stream)
    for _ in range(50):
        scene.replay(edit=True)
    ee[1].record(stream)
    torch.cuda.synchronize()
    edit_ms = ee[0].elapsed_time(ee[1]) / 50
    relight_only = []
    rr = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    rr[0].record(stream)
    for _ in range(20):
        scene.replay(edit=False)
    rr[1].record(stream)
    torch.cuda.synchronize()
    relight_ms = rr[0].elapsed_time(rr[1]) / 20

    cpu = None
    if rank == 0 and ws == 1 and not a.no_cpu_baseline:
        cpu = cpu_baseline(cfg, scene, dt, g, b, faces, mats, a.cpu_frames)
    secondary = None
    if rank == 0 and not a.no_secondary and a.side is None:
        # the other §8 rows, measured in the same run on the same GPU: the C2
        # medium interactive sequence (BASELINE configs[1]), the C4 sweep
        # (HBM-write roofline) and the C5 exact dipole precompute (FP32/SFU)
        del scene
        torch.cuda.empty_cache()
        sys.path.insert(0, str(ROOT / "tools"))
        import c2_bench
        import c5_bench
        import sweep_bench

        c2 = c2_bench.measure(100)
        torch.cuda.empty_cache()
        c4 = sweep_bench.measure(256, 20)
        c5 = c5_bench.measure(256)
        secondary = {
            "c2_medium_interactive": {k: c2[k] for k in (
                "points", "frames", "operator_nnz", "device_ms_per_frame", "device_points_per_s",
                "api_ms_per_frame", "api_points_per_s", "frame")},
            "c4_batched_sweep": {"kernel": "k_sweep_umma (tcgen05 bf16 UMMA, fp32 TMEM accum)",
                                 "us": c4["sweep_gemm_us"], "achieved_GBps": c4["achieved_GBps"],
                                 "peak_GBps": c4["peak_GBps"], "frac": c4["frac"],
                                 "bound": "hbm (fp32 output write)", "materials": c4["materials"],
                                 "K": c4["K"]},
            "c5_dipole_precompute": {
                "kernel": "k_pair_rows_exact (K-fused: R_d once per pair for all 8 terms, "
                          "receiver-tile blocks, + per-row top-2 % step 1)",
                "pairs": c5["pairs"], "materials": c5["materials"], "K": c5["K"],
                "pair_pass_s": c5["pair_pass_s"], "step1_select_s": c5["step1_select_s"],
                "pairs_per_s": c5["pairs_per_s"],
                "algorithmic_tflops": c5["algorithmic_tflops"],
                "fp32_peak_tflops": c5["fp32_peak_tflops"], "fp32_frac": c5["fp32_frac"],
                "flop_per_pair": 2000, "bound": "MUFU (4 per pair and material) / FP32"}}
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded geometry image + log-normal/lobe cubemap; BASELINE C3 shapes)",
            "config": workload_config(cfg, n, dt.nnz, ws),
            "setup": {"operator_bytes": dt.nbytes, "precompute_s": stats.get("precompute_s"),
                      "precompute_pairs": stats.get("pairs")},
            "roofline": {"bound": "hbm", "kernel": f"transfer[{kname}]",
                         "achieved": achieved,
                         "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "alg_bytes_per_launch": alg_bytes, "stored_bytes_per_launch": all_bytes,
                         "touched_nnz": touched, "kernel_ms": k_ms,
                         "kernel_choice_us": kchoice},
            "e2e": e2e,
            # per relight: env_project, env_irradiance, select (writes the packed x
            # and the kept bitmap), weights, transfer, edit_finish; per edit:
            # weights, edit_finish
            "gpu_launches": 6 * a.steps + 2 * n_edit,
            "clocks": clk,
            "relight_ms": relight_ms, "edit_ms": edit_ms,
            "cpu_baseline": cpu,
            "secondary": secondary,
        }
        print(json.dumps(line))
    if ws > 1:
        torch.distributed.destroy_process_group()


def _reference_ops(ops):
    """Reference-format operators (ours) -> the reference's own TransferOperator."""
    from oracle.reference_frame import import_reference

    R = import_reference()
    return [R["transfer"].TransferOperator(cols=o.cols, colptr=o.colptr, rowidx=o.rowidx,
                                           vals=o.vals, kept_energy=o.kept_energy,
                                           total_energy=o.total_energy,
                                           step1_entries=o.step1_entries) for o in ops]


def _reference_basis(b):
    from oracle.reference_frame import import_reference

    R = import_reference()
    return R["basisgen"].DiffusionBasis(r_nodes=b.r_nodes, bases=b.bases,
                                        singular_values=b.singular_values, eta=b.eta, g=b.g,
                                        sigma_box=tuple(b.sigma_box))


def _material_tuple(m):
    return (np.asarray(m.sigma_s_prime, np.float64), np.asarray(m.sigma_a, np.float64), float(m.eta))


def cpu_baseline(cfg, scene, dt, g, b, faces, mats, frames):
    """The reference's own frame (oracle/reference_frame.py: sssrelight from
    baseline/_ref, numba csc_apply on every host core) on `frames` frames of
    the bench sequence, operator from this run's GPU precompute. Returns the
    cpu_baseline object."""
    from oracle.reference_frame import ReferenceFrame, time_sequence

    cores = os.cpu_count() or 1
    t0 = time.perf_counter()
    ops = _reference_ops(dt.to_reference())
    fr = ReferenceFrame(ops, _reference_basis(b), g.positions, g.normals, cfg.side, cfg.levels,
                        cfg.e_keep, cfg.env_side, scene.camera.position, workers=cores)
    setup_s = time.perf_counter() - t0
    try:
        times = time_sequence(fr, faces, {f: _material_tuple(m) for f, m in mats.items()},
                              warmup=1, steps=frames, material0=_material_tuple(scene.material))
    finally:
        fr.close()
    per_frame = float(np.mean(times))
    return {"value": g.count / per_frame, "unit": UNIT, "cores": cores, "kind": "reference",
            "ms_per_step": per_frame * 1e3,
            "sample": f"{frames} whole C3 frames (after 1 warm-up) of the bench sequence through "
                      f"the reference's own code (baseline/_ref sssrelight: TransferOperator.apply "
                      f"= numba csc_apply, K x 3 calls over {cores} processes; compress_top_n, "
                      f"project_material, fresnel_transmittance) with the oracle's L-level Haar "
                      f"and environment-irradiance restatements; operator from this run's GPU "
                      f"precompute; setup {setup_s:.1f} s untimed"}


def export_operator(a, cfg, path):
    """Reference arm, step 1 (its own process, on the GPU): build the C3
    operator with this framework and write it as a PRTS1 container (the
    reference's on-disk format) + the frame inputs, so the timing process
    never maps this framework's library."""
    import torch

    from paper_2203_12339_b200 import _lib
    from paper_2203_12339_b200 import lighting as LT
    from paper_2203_12339_b200.basis import build_basis
    from paper_2203_12339_b200.geometry import make_geometry_image
    from paper_2203_12339_b200.precompute import precompute_compressed
    from paper_2203_12339_b200.prts1 import save_prts1

    _lib.load()
    g = make_geometry_image(cfg.side, cfg.radius, cfg.bump_amp, cfg.bump_terms, cfg.seed)
    b = build_basis(cfg.K, cfg.lattice)
    dt = precompute_compressed(g, b, cfg.levels, cfg.step1_keep, cfg.step2_fraction)
    torch.cuda.synchronize()
    save_prts1(path, b, dt.to_reference(), cfg.step1_keep, cfg.step2_fraction, cfg.side,
               mesh_hash=bytes(32), metadata={"config": cfg.name, "levels": cfg.levels})
    env = LT.Environment(side=cfg.env_side, seed=7)
    faces, mats = frame_inputs(cfg, env, a.warmup + a.steps, 100)
    from paper_2203_12339_b200.basis import OpticalMaterial
    from paper_2203_12339_b200.config import CAMERA

    m0 = OpticalMaterial(sigma_s_prime=cfg.material[0], sigma_a=cfg.material[1], eta=cfg.material[2])
    edit_frames = sorted(mats)
    np.savez(str(path) + ".inputs.npz", positions=g.positions, normals=g.normals,
             faces=np.stack(faces), edit_frames=np.array(edit_frames, np.int64),
             edit_mats=np.array([np.concatenate([mats[f].sigma_s_prime, mats[f].sigma_a,
                                                 [mats[f].eta]]) for f in edit_frames]).reshape(-1, 7),
             material0=np.concatenate([m0.sigma_s_prime, m0.sigma_a, [m0.eta]]),
             camera=np.array(CAMERA[0]), nnz=dt.nnz)


def run_reference(a, cfg):
    """--impl reference: the reference's own implementation of the C3 frame
    on this box's host cores (oracle/reference_frame.py), whole frames of the
    same sequence as ours. Step 1 (a separate GPU process) exports this run's
    operator as PRTS1; this process loads it with the reference's own loader
    and never imports the framework or maps its library."""
    ws, rank, local = _dist()
    if rank != 0:
        return
    from oracle.reference_frame import (ReferenceFrame, import_reference, load_reference_container,
                                        time_sequence)

    path = Path("/tmp") / f"sss_ref_{cfg.name}_{os.getpid()}.prts"
    t0 = time.perf_counter()
    env = dict(os.environ, CUDA_VISIBLE_DEVICES=os.environ.get("CUDA_VISIBLE_DEVICES", str(local)))
    res = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--config", a.config,
                          "--steps", str(a.steps), "--warmup", str(a.warmup),
                          "--export-operator", str(path)], env=env, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("reference arm: operator export failed")
    export_s = time.perf_counter() - t0
    R = import_reference()
    c = load_reference_container(path)
    z = np.load(str(path) + ".inputs.npz")
    cores = os.cpu_count() or 1
    fr = ReferenceFrame(c.compressed.operators, c.basis, z["positions"], z["normals"], cfg.side,
                        cfg.levels, cfg.e_keep, cfg.env_side, z["camera"], workers=cores)
    setup_s = time.perf_counter() - t0
    mats = {int(f): (m[0:3], m[3:6], float(m[6])) for f, m in zip(z["edit_frames"], z["edit_mats"])}
    m0 = z["material0"]
    try:
        times = time_sequence(fr, list(z["faces"]), mats, a.warmup, a.steps,
                              (m0[0:3], m0[3:6], float(m0[6])))
    finally:
        fr.close()
    for p in (path, Path(str(path) + ".inputs.npz")):
        try:
            p.unlink()
        except OSError:
            pass
    per_frame = float(np.mean(times))
    n = cfg.n
    loaded = sorted({Path(m.__file__).name for m in list(sys.modules.values())
                     if getattr(m, "__file__", None) and "paper_2203_12339_b200" in m.__file__})
    cpu = {"value": n / per_frame, "unit": UNIT, "cores": cores, "kind": "reference",
           "ms_per_step": per_frame * 1e3,
           "sample": f"{a.steps} whole C3 frames of the bench sequence (relight every frame, "
                     f"material edit every {cfg.extra.get('edit_every', 10)}) through the "
                     f"reference's own code ({R['backend']}: TransferOperator.apply = csc_apply, "
                     f"K x 3 calls over {cores} processes; compress_top_n, project_material, "
                     f"fresnel_transmittance) + the oracle's L-level Haar and environment "
                     f"irradiance restatements; operator loaded from a PRTS1 file by the "
                     f"reference's load_container (export {export_s:.1f} s, setup "
                     f"{setup_s:.1f} s, untimed)"}
    line = {"metric": METRIC, "value": cpu["value"], "unit": UNIT, "n_gpus": ws, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": cpu["ms_per_step"], "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "impl": "reference",
            "data": "synthetic (seeded geometry image + log-normal/lobe cubemap; BASELINE C3 shapes)",
            "config": workload_config(cfg, n, z["nnz"], ws),
            "cpu_baseline": cpu,
            "framework_modules_imported": loaded,
            "e2e": {"value": cpu["value"], "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def main():
    a = _args()
    from paper_2203_12339_b200.config import CONFIGS

    cfg = CONFIGS[a.config]
    if a.side:
        cfg = cfg.with_(side=a.side)
    if a.export_operator:
        export_operator(a, cfg, a.export_operator)
    elif a.impl == "reference":
        run_reference(a, cfg)
    else:
        run_ours(a, cfg)


if __name__ == "__main__":
    main()
