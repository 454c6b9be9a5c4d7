for l in base mf; do TP_LIBRARY=$PWD/exp_libs/$l.so timeout 300 python tools/dev/hash_out.py c5,c3,c4,c4b,c2,c1 0; done > gpurun_out/ab8_hash.log 2>&1
grep -v Warn gpurun_out/ab8_hash.log
timeout 1200 python tools/dev/ab_p1.py exp_libs/base.so,exp_libs/mf.so c5 p1ph,fullph 2 > gpurun_out/ab8_c5.log 2>&1
timeout 1200 python tools/ab_libs.py --libs exp_libs/base.so,exp_libs/mf.so --configs c3,c4,c4b,c2 --rounds 3 > gpurun_out/ab8_libs.log 2>&1
grep -v Warn gpurun_out/ab8_c5.log; cat gpurun_out/ab8_libs.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/ab8_gputest.log 2>&1; tail -5 gpurun_out/ab8_gputest.log
