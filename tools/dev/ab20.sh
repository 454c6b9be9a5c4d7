timeout 1200 python tools/dev/ab_p1.py exp_libs/chunk.so,exp_libs/k16.so,exp_libs/k32.so c5 p1ph,fullph 3 > gpurun_out/ab20_c5.log 2>&1
grep -v Warn gpurun_out/ab20_c5.log
