timeout 1200 python tools/dev/ab_p1.py exp_libs/base.so,exp_libs/deg3.so,exp_libs/notree.so,exp_libs/both.so c5 p1ph,fullph 2 > gpurun_out/ab5_c5.log 2>&1
grep -v Warn gpurun_out/ab5_c5.log
