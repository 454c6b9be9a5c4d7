for l in ctr3; do TP_LIBRARY=$PWD/exp_libs/$l.so timeout 300 python tools/dev/hash_out.py c5,c3 5; done > gpurun_out/ab24_hash.log 2>&1
grep -v Warn gpurun_out/ab24_hash.log
timeout 1200 python tools/dev/ab_p1.py exp_libs/cur2.so,exp_libs/ctr3.so c5 p1ph,fullph 3 > gpurun_out/ab24_c5.log 2>&1
grep -v Warn gpurun_out/ab24_c5.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/ab24_gputest.log 2>&1; tail -2 gpurun_out/ab24_gputest.log
timeout 400 python tools/soak.py --minutes 4 --seed 13 > gpurun_out/ab24_soak.log 2>&1; tail -1 gpurun_out/ab24_soak.log
