for l in sa3 sa4 sa5; do TP_LIBRARY=$PWD/exp_libs/$l.so timeout 300 python tools/dev/hash_out.py c4,c4b 0; done > gpurun_out/ab14_hash.log 2>&1
grep -v Warn gpurun_out/ab14_hash.log
timeout 1200 python tools/ab_libs.py --libs exp_libs/sa3.so,exp_libs/sa4.so,exp_libs/sa5.so --configs c4,c4b --rounds 3 > gpurun_out/ab14_libs.log 2>&1
cat gpurun_out/ab14_libs.log
