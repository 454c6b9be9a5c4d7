timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r23_gputest.log 2>&1; tail -2 gpurun_out/r23_gputest.log
timeout 400 python tools/soak.py --minutes 3 --seed 24 > gpurun_out/r23_soak.log 2>&1; tail -1 gpurun_out/r23_soak.log
for a in 2 3; do timeout 900 python tools/ab_libs.py --libs exp_libs/cur.so,exp_libs/cl3c.so --configs c4b,c4 --rounds 3 --reps 10 --algo $a --schedule 3; done > gpurun_out/r23.log 2>&1
