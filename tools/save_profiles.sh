#!/bin/bash
# Copy one evidence capture (tools/profile_round2.sh <tag>, merged into gpurun_out/) into profiles/:
# the bench line, the launch list, consecutive-call DRAM traffic (and profiles/traffic.json),
# ncu --set full summaries and per-line stall samples of C5 and C4b.
set -eu
tag=$1
tail -1 gpurun_out/${tag}_bench.log > profiles/${tag}_bench_c5.json
cp gpurun_out/${tag}_launches_bench.csv profiles/${tag}_launches_bench_c5.csv
cp gpurun_out/${tag}_traffic_*.csv profiles/
python tools/traffic.py $tag --out profiles/traffic.json > /dev/null
for c in c5 c4b; do
  python tools/ncu_summary.py gpurun_out/${tag}_full_$c.ncu-rep > profiles/${tag}_ncu_full_$c.json
  python tools/ncu_lines.py gpurun_out/${tag}_full_$c.ncu-rep 30 > profiles/${tag}_ncu_lines_$c.txt
done
ls profiles | grep "^${tag}_"
