for l in base t8 t16 t32; do TP_LIBRARY=$PWD/exp_libs/$l.so timeout 300 python tools/dev/hash_out.py c5,c3 5; done > gpurun_out/ab9_hash.log 2>&1
grep -v Warn gpurun_out/ab9_hash.log
timeout 1200 python tools/dev/ab_p1.py exp_libs/mf.so,exp_libs/t8.so,exp_libs/t16.so,exp_libs/t32.so c5 p1ph,fullph 2 > gpurun_out/ab9_c5.log 2>&1
grep -v Warn gpurun_out/ab9_c5.log
