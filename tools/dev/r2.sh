for c in c4b c4; do timeout 200 python tools/prof_cl_timeline.py $c --json gpurun_out/r2_tl_$c.json; done > gpurun_out/r2_tl.log 2>&1
timeout 900 python tools/ab_libs.py --libs exp_libs/fifo.so,exp_libs/lead2.so --configs c4b,c4 --rounds 4 --reps 10 > gpurun_out/r2_ab.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2_gputest.log 2>&1; tail -2 gpurun_out/r2_gputest.log
