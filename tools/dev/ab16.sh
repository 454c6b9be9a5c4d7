for l in cur prmt; do TP_LIBRARY=$PWD/exp_libs/$l.so timeout 300 python tools/dev/hash_out.py c4b 0; done > gpurun_out/ab16_hash.log 2>&1
grep -v Warn gpurun_out/ab16_hash.log
timeout 1200 python tools/ab_libs.py --libs exp_libs/cur.so,exp_libs/prmt.so --configs c4b --rounds 4 > gpurun_out/ab16_libs.log 2>&1
cat gpurun_out/ab16_libs.log
