for l in lean npf; do TP_LIBRARY=$PWD/exp_libs/$l.so timeout 300 python tools/dev/hash_out.py c4,c4b,c3 0; done > gpurun_out/ab12_hash.log 2>&1
grep -v Warn gpurun_out/ab12_hash.log
timeout 1200 python tools/ab_libs.py --libs exp_libs/lean.so,exp_libs/npf.so --configs c3,c4,c4b --rounds 3 > gpurun_out/ab12_libs.log 2>&1
cat gpurun_out/ab12_libs.log
