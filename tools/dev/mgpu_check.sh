# functional check of bench.py's N = 2 paths with both ranks on the one GPU (gloo; not a measurement).
# nvlink-fused cannot run this way: its finish kernel waits in-kernel for the other rank's
# partial kernel, and two processes on one GPU are time-sliced (the watchdog fires).
export TP_BENCH_ONE_DEVICE=1 TP_BENCH_BACKEND=gloo
for ex in ${EXCH:-nccl nvlink}; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29533 \
    bench.py --gpus 2 --steps 3 --warmup 3 --exchange $ex --also c4 > gpurun_out/mg_$ex.log 2>&1
  echo "== $ex rc=$?"; tail -1 gpurun_out/mg_$ex.log | cut -c1-600
done
