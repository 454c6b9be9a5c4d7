#!/bin/bash
# A/B timing of two library builds in one gpurun call: bash tools/ab.sh <libB.so> <stress specs...>
B=$1; shift
for i in 1 2; do
  echo "== A (libtwopass.so)"; timeout 300 python tools/stress.py "$@" --reps 20 | python -c "import sys,json;[print(json.loads(l)['spec'], round(json.loads(l)['median_us'],1)) for l in sys.stdin if l.startswith('{')]"
  echo "== B ($B)"; TP_LIBRARY=$PWD/paper_2001_04438_b200/$B timeout 300 python tools/stress.py "$@" --reps 20 | python -c "import sys,json;[print(json.loads(l)['spec'], round(json.loads(l)['median_us'],1)) for l in sys.stdin if l.startswith('{')]"
done
