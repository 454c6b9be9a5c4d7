for l in chunk2; do TP_LIBRARY=$PWD/exp_libs/$l.so timeout 300 python tools/dev/hash_out.py c5,c3,c2 0; done > gpurun_out/ab21_hash.log 2>&1
grep -v Warn gpurun_out/ab21_hash.log
timeout 1200 python tools/dev/ab_p1.py exp_libs/chunk.so,exp_libs/chunk2.so c5 p1ph,fullph 3 > gpurun_out/ab21_c5.log 2>&1
timeout 1200 python tools/dev/ab_p1.py exp_libs/chunk.so,exp_libs/chunk2.so c3 p1st,fullst,p1ph,fullph 3 >> gpurun_out/ab21_c5.log 2>&1
grep -v Warn gpurun_out/ab21_c5.log
python tools/prof_phase.py c5 --reps 3 2>&1 | head -8; python tools/prof_phase.py c3 --reps 3 2>&1 | head -8
