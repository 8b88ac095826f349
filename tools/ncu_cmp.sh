#!/bin/bash
# ncu one mid-circuit pass under a given timing-experiment mode; print key metrics
M=$1
ncu --set full --clock-control none -k regex:svpass -s 11 -c 1 -o /tmp/cmp_$M python tools/exp_timing.py $M > /dev/null 2>&1
ncu -i /tmp/cmp_$M.ncu-rep --page details --csv > /tmp/cmp_$M.csv
python tools/ncu_summary.py details /tmp/cmp_$M.csv | grep -E "Duration|Shared Memory Configuration|Block Limit|L1/TEX Hit|L2 Hit|Achieved Occupancy|Issue Slots|Executed Instructions |Mem Busy|Max Bandwidth|Registers" | sed "s/^/[$M] /"
