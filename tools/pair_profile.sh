#!/bin/bash
# --set full captures of the pair kernels of the 30 q c64 plan (second run: launches 5 and 8)
O=gpurun_out/${1:-pair_prof}
mkdir -p $O
for spec in 5:p01 8:p45; do
  IFS=: read skip tag <<< "$spec"
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:svpass -s $skip -c 1 -o /tmp/pair_$tag \
      python tools/run_plan.py --dtype c64 > $O/run_$tag.log 2>&1
  ncu -i /tmp/pair_$tag.ncu-rep --page details --csv > $O/pair_${tag}_details.csv
  ncu -i /tmp/pair_$tag.ncu-rep --page raw --csv > $O/pair_${tag}_raw.csv
  cp /tmp/pair_$tag.ncu-rep $O/
done
