#!/bin/bash
set -u
out=gpurun_out; mkdir -p $out
for spec in "c4b rowcl 2" "c4 rowcl 2" "c5 rowph 1"; do
  set -- $spec
  timeout 120 python tools/prof_run.py --config $1 --iters 2 > $out/s_plain_$1.log 2>&1 || continue
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$2 -s $3 -c 1 \
    -o $out/s_full_$1 python tools/prof_run.py --config $1 --iters 2 > $out/s_ncu_$1.log 2>&1
  ncu -i $out/s_full_$1.ncu-rep --page source --csv --print-source sass > $out/s_src_$1.csv 2>/dev/null
  ncu -i $out/s_full_$1.ncu-rep --page source --csv --print-source cuda > $out/s_cuda_$1.csv 2>/dev/null
done
ls -la $out
