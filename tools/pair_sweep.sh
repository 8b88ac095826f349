#!/bin/bash
# pair kernels: per-pass device times (tools/run_plan.py) vs SV_PAIR_WAVES / SV_PAIR_LOOK, and without pairing
O=gpurun_out/${1:-pair_sweep}
mkdir -p $O
for dt in c64 c128; do
  echo "== $dt SV_PAIR=0" >> $O/sweep.txt
  SV_PAIR=0 timeout 300 python tools/run_plan.py --dtype $dt 2>&1 | grep "pass ms" >> $O/sweep.txt
  for w in 0.5 1; do for l in 1 2 3; do
    echo "== $dt waves $w look $l" >> $O/sweep.txt
    SV_PAIR_LOOK=$l SV_PAIR_WAVES=$w timeout 300 python tools/run_plan.py --dtype $dt 2>&1 | grep "pass ms" >> $O/sweep.txt
  done; done
done
cat $O/sweep.txt
