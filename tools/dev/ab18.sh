for l in phi phs8 phs4; do echo "== $l"; TP_LIBRARY=$PWD/exp_libs/$l.so timeout 300 python tools/dev/ph_sweep.py c4,c4b 16,24,32,48; done > gpurun_out/ab18.log 2>&1
grep -v Warn gpurun_out/ab18.log | grep -v auto
