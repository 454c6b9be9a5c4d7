for l in acq; do TP_LIBRARY=$PWD/exp_libs/$l.so timeout 300 python tools/dev/hash_out.py c5,c3 0; TP_LIBRARY=$PWD/exp_libs/$l.so timeout 300 python tools/dev/hash_out.py c3 5; done > gpurun_out/ab15_hash.log 2>&1
grep -v Warn gpurun_out/ab15_hash.log
timeout 1200 python tools/dev/ab_p1.py exp_libs/fences.so,exp_libs/acq.so c3 p1ph,fullph,p1st,fullst 3 > gpurun_out/ab15_c3.log 2>&1
timeout 1200 python tools/dev/ab_p1.py exp_libs/fences.so,exp_libs/acq.so c5 fullph 2 >> gpurun_out/ab15_c3.log 2>&1
grep -v Warn gpurun_out/ab15_c3.log
