#!/bin/bash
O=gpurun_out/${1:-rt}
mkdir -p $O
for r in 1 2; do
for v in 0 1; do
  echo "== SV_RT_SCALAR=$v rep $r" >> $O/rt.txt
  for dt in c64 c128; do SV_RT_SCALAR=$v timeout 300 python tools/run_plan.py --dtype $dt 2>&1 | grep "pass ms" >> $O/rt.txt; done
done; done
cat $O/rt.txt
