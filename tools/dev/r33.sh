timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "host" > gpurun_out/r33_tests.log 2>&1; tail -2 gpurun_out/r33_tests.log
timeout 900 python bench.py --also "" --no-three-pass > gpurun_out/r33_bench.log 2>&1; tail -1 gpurun_out/r33_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps(d['e2e'])); print(d['ms_per_step'])"
