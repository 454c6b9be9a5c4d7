set -u
mkdir -p gpurun_out
for l in base h4 h5 h7; do echo "== $l"; TP_LIBRARY=$PWD/exp_libs/$l.so timeout 120 python tools/dev/hash_out.py c3 5 2>&1 | grep -v Warn | tail -2; done > gpurun_out/ab3.log 2>&1
TP_LIBRARY=$PWD/exp_libs/h7.so timeout 300 compute-sanitizer --tool memcheck python tools/dev/hash_out.py c3 5 > gpurun_out/ab3_san.log 2>&1
cat gpurun_out/ab3.log; head -60 gpurun_out/ab3_san.log
