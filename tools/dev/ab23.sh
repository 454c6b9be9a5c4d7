for l in ctr2; do TP_LIBRARY=$PWD/exp_libs/$l.so timeout 300 python tools/dev/hash_out.py c4,c4b 0; done > gpurun_out/ab23_hash.log 2>&1
grep -v Warn gpurun_out/ab23_hash.log
timeout 1200 python tools/ab_libs.py --libs exp_libs/cur2.so,exp_libs/ctr2.so --configs c4,c4b,c5 --rounds 3 > gpurun_out/ab23_libs.log 2>&1
cat gpurun_out/ab23_libs.log
