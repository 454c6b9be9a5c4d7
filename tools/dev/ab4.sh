mkdir -p gpurun_out
TP_LIBRARY=$PWD/exp_libs/h7.so timeout 300 python tools/dev/h7probe.py 29,30,31 c5 > gpurun_out/ab4.log 2>&1
grep -v Warn gpurun_out/ab4.log | tail -30
