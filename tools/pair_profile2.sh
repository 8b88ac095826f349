#!/bin/bash
O=gpurun_out/${1:-pair_prof2}
mkdir -p $O
timeout 600 ncu --set full --clock-control none -k regex:svpass -s 8 -c 1 -o /tmp/pair_p45 python tools/run_plan.py --dtype c64 > /dev/null 2>&1
for spec in 11:s4 12:s5 7:s0; do
  IFS=: read skip tag <<< "$spec"
  SV_PAIR=0 timeout 600 ncu --set full --clock-control none -k regex:svpass -s $skip -c 1 -o /tmp/single_$tag python tools/run_plan.py --dtype c64 > /dev/null 2>&1
done
cp /tmp/pair_p45.ncu-rep /tmp/single_*.ncu-rep $O/
