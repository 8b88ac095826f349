#!/bin/bash
# Round-3 captures (run under gpurun): --set full of c64 passes 0 (basis variant), 2, 3 and c128
# pass 3 of the second run of the plan; raw + details CSV exported for tools/ncu_summary.py.
R=${1:-late}
OUT=gpurun_out/profile_$R
mkdir -p $OUT
for spec in c64:7:p0 c64:9:p2 c64:10:p3 c128:10:p3; do
  IFS=: read dt skip tag <<< "$spec"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:svpass -s $skip -c 1 -o /tmp/full_${dt}_$tag \
      python tools/run_plan.py --dtype $dt > /dev/null 2>&1
  ncu -i /tmp/full_${dt}_$tag.ncu-rep --page details --csv > $OUT/full_${dt}_supremacy_${tag}_details.csv
  ncu -i /tmp/full_${dt}_$tag.ncu-rep --page raw --csv > $OUT/full_${dt}_supremacy_${tag}_raw.csv
  ncu -i /tmp/full_${dt}_$tag.ncu-rep --page source --csv --print-source sass > $OUT/full_${dt}_supremacy_${tag}_sass.csv 2>&1
done
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > $OUT/gpu.txt
