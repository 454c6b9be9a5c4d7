#!/bin/bash
# Evidence capture for profiles/ (run under gpurun from the repo root; one GPU).
#   bash tools/profile_round.sh <tag>
# 1. the bench command runs plain, then again under ncu for the launch list (device time and
#    DRAM bytes per launch; cold-cache serialised: compare shares, not absolutes);
# 2. one ncu --set full capture of each headline kernel (C4 cluster, C4b cluster, C3 stream).
set -u
tag=${1:-r01}
out=gpurun_out
mkdir -p $out
timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e > $out/${tag}_bench_plain.log 2>&1 || exit 1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file $out/${tag}_launches_bench_c4.csv python bench.py --steps 3 --warmup 3 --no-e2e > $out/${tag}_ncu_launches.log 2>&1
# (skip counts: a cluster launch is followed by its concurrent side launch of the same kernel,
# so the second matching launch is the side one; -s 2 captures the second call's main launch)
for spec in "c4 0 rowcl 2" "c4b 0 rowcl 2" "c3 0 stream_kernel 1" "c2 0 small_kernel 1"; do
  set -- $spec
  timeout 120 python tools/prof_run.py --config $1 --iters 2 --schedule $2 > $out/${tag}_plain_$1.log 2>&1 || continue
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:$3 -s $4 -c 1 \
    -o $out/${tag}_full_$1 python tools/prof_run.py --config $1 --iters 2 --schedule $2 > $out/${tag}_ncu_full_$1.log 2>&1
done
echo profile_round done
