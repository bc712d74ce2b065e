"""Summaries under profiles/ from a gpurun capture directory:

* <prefix>_launches.csv          the raw ncu launch list (copied)
* <prefix>_launches_summary.csv  per-kernel launches / mean us / share of a relight frame
* <prefix>_transfer_dram_bytes.json  DRAM bytes, duration, throughput and stalls of the
                                 dominant kernel from one `ncu --set full` capture

    python tools/summarize_profiles.py gpurun_out/r01b --prefix r01 [--rep transfer_full.ncu-rep]
"""
import argparse
import csv
import json
import shutil
import subprocess
from collections import OrderedDict, defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
FRAME = ("k_transfer_kfr", "k_transfer_flat16", "k_transfer_flat8s", "k_env_irradiance_multi", "k_env_irradiance_chan", "k_select_cluster", "k_env_project",
         "k_edit_finish_multi", "k_material_weights", "k_env_union", "k_pack_x_bits",
         "k_sh_irradiance_multi", "k_direct_single", "k_fold_apply_rows")
METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "dram__throughput.avg.pct_of_peak_sustained_elapsed",
           "l1tex__throughput.avg.pct_of_peak_sustained_active",
           "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
           "lts__throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
           "smsp__issue_active.avg.pct_of_peak_sustained_active", "l1tex__t_sector_hit_rate.pct",
           "launch__registers_per_thread", "launch__grid_size", "launch__block_size"]


def launches(src: Path, prefix: str, out: Path):
    rows = [r for r in csv.reader(open(src)) if len(r) > 5]
    h = rows[0]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    t = defaultdict(list)
    for r in rows[1:]:
        name = r[ki].split("(")[0].replace("void ", "").strip()
        scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}
        t[name].append(float(r[vi].replace(",", "")) * scale.get(r[ui], 1e-3))
    frame = OrderedDict((k, v) for k, v in sorted(t.items(), key=lambda kv: -sum(kv[1]))
                        if any(f in k for f in FRAME))
    setup = OrderedDict((k, v) for k, v in sorted(t.items(), key=lambda kv: -sum(kv[1]))
                        if k not in frame)
    relight = sum(sum(v) / len(v) for k, v in frame.items()
                  if "k_edit_finish" not in k and "k_material_weights" not in k)
    relight += sum(sum(v) / len(v) for k, v in frame.items() if "k_edit_finish" in k)
    lines = [f"# {prefix} ncu launch list summary (gpu__time_duration.sum, --clock-control none; "
             "cold-cache, serialized)",
             f"# source: profiles/{prefix}_launches.csv (ncu --nvtx --nvtx-include timed/ python "
             "bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-secondary: the timed frames only)",
             "# --- per-frame kernels (relight; edit frames: k_material_weights + k_edit_finish_multi)",
             "kernel,launches,mean_us,share_of_relight_pct"]
    for k, v in frame.items():
        m = sum(v) / len(v)
        share = "" if "k_material_weights" in k else f"{100 * m / relight:.1f}"
        lines.append(f"{k},{len(v)},{m:.2f},{share}")
    lines.append(f"# relight kernel sum: {relight:.1f} us (material weights run on a forked "
                 "stream inside the graph)")
    lines.append("# --- setup: GPU precompute of the C3 operator and tables")
    for k, v in setup.items():
        lines.append(f"{k},{len(v)},{sum(v) / len(v):.2f},")
    (out / f"{prefix}_launches_summary.csv").write_text("\n".join(lines) + "\n")
    shutil.copy(src, out / f"{prefix}_launches.csv")


def full(rep: Path, prefix: str, out: Path, command: str):
    raw = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    r = list(csv.reader(raw.splitlines()))
    h, u, v = r[0], r[1], r[2]
    kname = v[h.index("Kernel Name")] if "Kernel Name" in h else ""
    met = {k: [v[h.index(k)], u[h.index(k)]] for k in METRICS if k in h}
    stalls = sorted(((k, float(v[h.index(k)])) for k in h
                     if k.startswith("smsp__average_warps_issue_stalled_") and
                     k.endswith("_per_issue_active.ratio") and v[h.index(k)] not in ("", "n/a")),
                    key=lambda kv: -kv[1])[:8]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    rd = float(met["dram__bytes_read.sum"][0].replace(",", "")) * scale[met["dram__bytes_read.sum"][1]]
    wr = float(met["dram__bytes_write.sum"][0].replace(",", "")) * scale[met["dram__bytes_write.sum"][1]]
    js = {"kernel": kname[:90], "capture": command, "dram_bytes_per_launch": rd + wr,
          "dram_read_bytes": rd, "dram_write_bytes": wr, "metrics": met,
          "top_stalls_per_issue": stalls}
    kk = "kfr" if "kfr" in kname else ("flat16" if "flat16" in kname else "")
    name = f"{prefix}_transfer_{kk}_dram_bytes.json" if kk else f"{prefix}_transfer_dram_bytes.json"
    (out / name).write_text(json.dumps(js, indent=1) + "\n")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("src")
    ap.add_argument("--prefix", default="r01")
    ap.add_argument("--rep", default="transfer_full.ncu-rep")
    a = ap.parse_args()
    src = Path(a.src)
    out = ROOT / "profiles"
    if (src / "launches.csv").exists():
        launches(src / "launches.csv", a.prefix, out)
    if (src / a.rep).exists():
        full(src / a.rep, a.prefix, out, "ncu --set full --import-source on --clock-control none "
             "-k regex:k_transfer_kfr -s 3 -c 1, C3 bench (bench.py --steps 3 --warmup 3 "
             "--no-cpu-baseline --no-secondary)")


if __name__ == "__main__":
    main()
