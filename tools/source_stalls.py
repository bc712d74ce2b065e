"""Per-instruction warp-stall samples of one kernel from an `ncu --set full
--import-source on` capture (the source page): total samples by stall reason
and the SASS instructions that collect the most.

    python tools/source_stalls.py gpurun_out/r02f/transfer_full.ncu-rep profiles/r02_transfer_kfr_source_stalls.json
"""
import csv
import json
import subprocess
import sys


def main():
    rep, out = sys.argv[1], sys.argv[2]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    kernel = rows[0][1] if rows and len(rows[0]) > 1 else ""
    h, data = rows[1], rows[2:]
    ix = {n: i for i, n in enumerate(h)}
    stalls = [n for n in h if n.startswith("stall_") and "Not Issued" not in n]
    tot = sum(int(r[ix["# Samples"]]) for r in data)
    agg = {n: sum(int(r[ix[n]]) for r in data) for n in stalls}
    top = sorted(data, key=lambda r: -int(r[ix["# Samples"]]))[:25]
    res = {"capture": rep.split("/")[-1], "kernel": kernel[:80], "samples": tot,
           "by_reason_pct": {k: round(100 * v / tot, 1) for k, v in
                             sorted(agg.items(), key=lambda kv: -kv[1]) if v},
           "top_instructions": [
               {"sass": r[ix["Source"]].strip()[:70], "samples_pct": round(100 * int(r[ix["# Samples"]]) / tot, 2),
                "executed": int(r[ix["Instructions Executed"]]),
                "reasons": dict(sorted(((n, int(r[ix[n]])) for n in stalls if int(r[ix[n]]) > 0),
                                       key=lambda kv: -kv[1])[:3])} for r in top]}
    with open(out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res["by_reason_pct"]))


if __name__ == "__main__":
    main()
