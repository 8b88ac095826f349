#!/bin/bash
# heavy passes (one register bit fewer): resident warps per SM (SV_MIN_WARPS_HEAVY)
O=gpurun_out/${1:-heavy}
mkdir -p $O
for r in 1 2; do
for w in 0 24 32; do
  echo "== SV_MIN_WARPS_HEAVY=$w rep $r" >> $O/heavy.txt
  for dt in c64 c128; do SV_MIN_WARPS_HEAVY=$w timeout 300 python tools/run_plan.py --dtype $dt 2>&1 | grep "pass ms" >> $O/heavy.txt; done
done; done
cat $O/heavy.txt
