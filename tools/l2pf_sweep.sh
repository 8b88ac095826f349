#!/bin/bash
O=gpurun_out/${1:-l2pf}
mkdir -p $O
for r in 1 2; do for d in 0 370 740 1480; do
  echo "== SV_L2PF=$d rep $r" >> $O/l2pf.txt
  for dt in c64 c128; do SV_L2PF=$d timeout 300 python tools/run_plan.py --dtype $dt 2>&1 | grep "pass ms" >> $O/l2pf.txt; done
done; done
cat $O/l2pf.txt
