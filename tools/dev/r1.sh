set -x
for c in c4b c4; do
  for l in base fifo; do TP_LIBRARY=$PWD/exp_libs/$l.so timeout 200 python tools/prof_roles.py $c --reps 5; done
done > gpurun_out/r1_roles.log 2>&1
timeout 900 python tools/ab_libs.py --libs exp_libs/base.so,exp_libs/fifo.so --configs c4b,c4 --rounds 5 --reps 10 > gpurun_out/r1_ab.log 2>&1
