#!/bin/bash
# A/B per-pass times of the 30 q supremacy plans under environment variants (run under gpurun).
# usage: tools/ab_env.sh OUTDIR "ENV1" "ENV2" ...   ("-" = no extra environment)
O=gpurun_out/$1; shift; mkdir -p $O
for rep in 1 2; do
for v in "$@"; do
  for dt in c64 c128; do
    r=$(env ${v/#-/} timeout 300 python tools/run_plan.py --dtype $dt 2>&1 | tail -1)
    echo "[$dt] $v: $r" >> $O/ab.txt
  done
done
done
cat $O/ab.txt
