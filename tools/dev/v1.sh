timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/v1_gputest.log 2>&1; tail -3 gpurun_out/v1_gputest.log
timeout 400 python tools/soak.py --minutes 5 --seed 11 > gpurun_out/v1_soak.log 2>&1; tail -3 gpurun_out/v1_soak.log
timeout 900 python bench.py > gpurun_out/v1_bench.log 2>&1; tail -1 gpurun_out/v1_bench.log | cut -c1-300
