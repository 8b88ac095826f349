#!/bin/bash
# small-state latency under register-width variants (run under gpurun)
O=gpurun_out/${1:-small_rb}; mkdir -p $O
for v in - SV_RB=4 SV_RB=3 SV_RB=2; do
  env ${v/#-/} timeout 300 python tools/small_lat.py >> $O/lat.txt 2>&1
done
cat $O/lat.txt
