"""Key ncu metrics of the frame's stage-1 / epilogue kernels from `ncu --set
full` captures (one launch each): duration, DRAM bytes and throughput, pipe
and issue utilisation, top stalls.

    python tools/chain_ncu_summary.py gpurun_out/r02f/chain_*.ncu-rep > profiles/r02_chain_ncu.json
"""
import csv
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__cluster_size"]


def main():
    out = {}
    for rep in sys.argv[1:]:
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                             text=True).stdout
        r = list(csv.reader(raw.splitlines()))
        if len(r) < 3:
            continue
        h, u, v = r[0], r[1], r[2]
        name = v[h.index("Kernel Name")].split("(")[0].replace("void ", "").replace("sss::", "")
        met = {k: f"{v[h.index(k)]} {u[h.index(k)]}".strip() for k in KEYS if k in h}
        stalls = sorted(((k.replace("smsp__average_warps_issue_stalled_", "").replace(
            "_per_issue_active.ratio", ""), float(v[h.index(k)])) for k in h
            if k.startswith("smsp__average_warps_issue_stalled_") and
            k.endswith("_per_issue_active.ratio") and v[h.index(k)] not in ("", "n/a")),
            key=lambda kv: -kv[1])[:5]
        out[name] = {"metrics": met, "top_stalls_per_issue": dict(stalls)}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
