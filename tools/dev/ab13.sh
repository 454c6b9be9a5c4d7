for l in team8 team10 team12; do TP_LIBRARY=$PWD/exp_libs/$l.so timeout 300 python tools/dev/hash_out.py c4,c4b 0; done > gpurun_out/ab13_hash.log 2>&1
grep -v Warn gpurun_out/ab13_hash.log
timeout 1200 python tools/ab_libs.py --libs exp_libs/lean.so,exp_libs/team8.so,exp_libs/team10.so,exp_libs/team12.so --configs c4,c4b --rounds 3 > gpurun_out/ab13_libs.log 2>&1
cat gpurun_out/ab13_libs.log
