set -x
for lib in libtwopass.so libtwopass_st1.so libtwopass_st2.so; do
 for h in 1 0 2 3; do
  echo "== lib=$lib hints=$h"
  TP_LIBRARY=$PWD/paper_2001_04438_b200/$lib TP_L2_HINTS=$h timeout 120 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:rowcl -c 2 python tools/prof_run.py --config c4 --iters 2 --schedule 3 2>&1 | grep -E "dram__|gpu__time" | tail -3
 done
done
