timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/v2_gputest.log 2>&1; tail -3 gpurun_out/v2_gputest.log
timeout 400 python tools/soak.py --minutes 5 --seed 12 > gpurun_out/v2_soak.log 2>&1; tail -3 gpurun_out/v2_soak.log
