for l in base defer; do TP_LIBRARY=$PWD/exp_libs/$l.so timeout 300 python tools/dev/hash_out.py c5,c3 5; done > gpurun_out/ab6_hash.log 2>&1
timeout 1200 python tools/dev/ab_p1.py exp_libs/base.so,exp_libs/defer.so c5 p1ph,fullph 3 > gpurun_out/ab6_c5.log 2>&1
timeout 1200 python tools/dev/ab_p1.py exp_libs/base.so,exp_libs/defer.so c3 p1ph,fullph,p1st,fullst 2 > gpurun_out/ab6_c3.log 2>&1
grep -v Warn gpurun_out/ab6_hash.log; grep -v Warn gpurun_out/ab6_c5.log gpurun_out/ab6_c3.log
