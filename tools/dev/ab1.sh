set -u
mkdir -p gpurun_out
for l in base h7 pf h7pf; do TP_LIBRARY=$PWD/exp_libs/$l.so timeout 300 python tools/dev/hash_out.py c5,c3 5; done > gpurun_out/ab1_hash.log 2>&1
timeout 1200 python tools/dev/ab_p1.py exp_libs/base.so,exp_libs/h7.so,exp_libs/pf.so,exp_libs/h7pf.so c5 p1ph,fullph 3 > gpurun_out/ab1_c5.log 2>&1
cat gpurun_out/ab1_hash.log gpurun_out/ab1_c5.log
