timeout 1200 python tools/dev/ab_p1.py exp_libs/lean.so c3 p1ph,fullph,p1st,fullst 3 > gpurun_out/ab11_c3.log 2>&1
grep -v Warn gpurun_out/ab11_c3.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/ab11_gputest.log 2>&1; tail -3 gpurun_out/ab11_gputest.log
timeout 900 python bench.py > gpurun_out/ab11_bench.log 2>&1; tail -1 gpurun_out/ab11_bench.log | cut -c1-400
