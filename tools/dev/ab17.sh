for l in la1 la2 la3; do TP_LIBRARY=$PWD/exp_libs/$l.so timeout 300 python tools/dev/hash_out.py c4,c4b 0; done > gpurun_out/ab17_hash.log 2>&1
grep -v Warn gpurun_out/ab17_hash.log
timeout 1200 python tools/ab_libs.py --libs exp_libs/la1.so,exp_libs/la2.so,exp_libs/la3.so --configs c4,c4b --rounds 3 > gpurun_out/ab17_libs.log 2>&1
cat gpurun_out/ab17_libs.log
