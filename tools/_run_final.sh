#!/bin/bash
# Final-state measurements of a round: bench (both arms), the ncu launch list of
# the timed frames, one full ncu capture of the transfer kernel, the graph
# timeline and the phase traces. Run on the GPU box: bash tools/_run_final.sh <dir>
D=${1:-gpurun_out/r02f}
mkdir -p $D
python bench.py > $D/bench.json 2> $D/bench.err
python bench.py --steps 1000 --warmup 5 --no-cpu-baseline --no-secondary > $D/bench_1000.json 2> $D/bench_1000.err
python bench.py --impl reference --steps 3 --warmup 1 > $D/bench_ref.json 2> $D/bench_ref.err
ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $D/launches.csv python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-secondary \
  > $D/ncu_launches.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_transfer_kfr -s 3 -c 1 -f \
  -o $D/transfer_full python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-secondary \
  > $D/ncu_full.log 2>&1
python tools/graph_timeline.py --out $D/timeline.json > $D/timeline.log 2>&1
python tools/env_trace.py 2>&1 | tail -1 > $D/env_trace.json
python tools/select_trace.py 2>&1 | tail -1 > $D/select_trace.json
python tools/e2e_breakdown.py 2>&1 | tail -1 > $D/e2e_breakdown.json
python tools/pcie_probe.py > $D/pcie_probe.txt 2>&1
ls -la $D
