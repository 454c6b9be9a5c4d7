#!/bin/bash
# Evidence capture for the C5 headline (run under gpurun from the repo root; one GPU).
#   bash tools/profile_c5.sh <tag>
# 1. bench.py on C5 (the driver's default command), plain;
# 2. the launch list of four back-to-back C5 calls with DRAM bytes per launch and NO cache
#    control (launch k's bytes then include the write-back of launch k-1's dirty L2 lines, so
#    launches 2..4 carry a whole step's DRAM traffic);
# 3. one `ncu --set full` capture of the second C5 launch (stream kernel).
set -u
tag=${1:-r02}
out=gpurun_out
mkdir -p $out
timeout 600 python bench.py --workload c5 --steps 20 --warmup 5 > $out/${tag}_bench_c5.log 2>&1 || { echo bench failed; exit 1; }
timeout 300 python tools/prof_run.py --config c5 --iters 4 > $out/${tag}_plain_c5.log 2>&1 || { echo plain failed; exit 1; }
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --cache-control none \
  --clock-control none --csv --log-file $out/${tag}_launches_c5.csv python tools/prof_run.py --config c5 --iters 4 \
  > $out/${tag}_ncu_launches_c5.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:stream_kernel -s 1 -c 1 \
  -o $out/${tag}_full_c5 python tools/prof_run.py --config c5 --iters 2 > $out/${tag}_ncu_full_c5.log 2>&1
echo profile_c5 done
