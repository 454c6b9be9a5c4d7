for l in ctr; do TP_LIBRARY=$PWD/exp_libs/$l.so timeout 300 python tools/dev/hash_out.py c5,c3 5; done > gpurun_out/ab22_hash.log 2>&1
grep -v Warn gpurun_out/ab22_hash.log
timeout 1200 python tools/dev/ab_p1.py exp_libs/cur2.so,exp_libs/ctr.so c5 p1ph,fullph 3 > gpurun_out/ab22_c5.log 2>&1
grep -v Warn gpurun_out/ab22_c5.log
