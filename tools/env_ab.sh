#!/bin/bash
# A/B of one environment knob on the 30 q plans (tools/run_plan.py per-pass times), 3 alternating repeats
# usage: tools/env_ab.sh OUTTAG VAR VALUE
O=gpurun_out/${1:-ab}; VAR=$2; VAL=$3
mkdir -p $O
for r in 1 2 3; do
  for v in 0 $VAL; do
    echo "== $VAR=$v rep $r" >> $O/ab.txt
    for dt in c64 c128; do env $VAR=$v timeout 300 python tools/run_plan.py --dtype $dt 2>&1 | grep "pass ms" >> $O/ab.txt; done
  done
done
cat $O/ab.txt
