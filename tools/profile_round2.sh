#!/bin/bash
# Round-2 evidence capture (run under gpurun from the repo root; one GPU):
#   bash tools/profile_round2.sh <tag>
# 1. bench.py as the driver runs it (plain), its JSON line kept;
# 2. the launch list of a short bench run (device time per launch: shares, not absolutes);
# 3. per workload, 4 consecutive calls with DRAM bytes and --cache-control none (tools/traffic.py);
# 4. one `ncu --set full` capture of C5's kernel (second call) and of C4b's cluster kernel.
set -u
tag=${1:-r02}
out=gpurun_out
mkdir -p $out
timeout 900 python bench.py > $out/${tag}_bench.log 2>&1 || { echo bench failed; tail -5 $out/${tag}_bench.log; exit 1; }
timeout 600 python bench.py --steps 2 --warmup 3 --no-e2e --also "" > $out/${tag}_bench_short.log 2>&1 &&
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/${tag}_launches_bench.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --also "" > $out/${tag}_ncu_launches.log 2>&1
for cfg in c5 c4 c4b c3 c2; do
  timeout 300 python tools/prof_run.py --config $cfg --iters 4 > $out/${tag}_plain_$cfg.log 2>&1 || continue
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --cache-control none \
    --clock-control none --csv --log-file $out/${tag}_traffic_$cfg.csv python tools/prof_run.py --config $cfg --iters 4 \
    > $out/${tag}_ncu_traffic_$cfg.log 2>&1
done
for spec in "c5 rowph 1" "c4b rowres 1"; do
  set -- $spec
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:$2 -s $3 -c 1 \
    -o $out/${tag}_full_$1 python tools/prof_run.py --config $1 --iters 2 > $out/${tag}_ncu_full_$1.log 2>&1
done
echo profile_round2 done
