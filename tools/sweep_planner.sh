#!/bin/bash
# planner knob sweep (commutation rule x pass budget) with per-pass event timing
DT=${1:-c64}
for cm in 0 1; do for b in 90 110 140 1000; do
  r=$(SV_COMMUTE=$cm SV_PASS_BUDGET=$b python tools/run_plan.py --dtype $DT 2>&1 | tail -1 | sed 's/.*total/total/')
  echo "[$DT] commute=$cm budget=$b $r"
done; done
