#!/bin/bash
# planner/kernel knob sweep on the 30q supremacy d20 plan: total device ms of the passes
# usage: tools/sweep_relabel.sh "c64:12 c64:13 c128:12" "16 20 24"
CFG="${1:-c64:11 c64:12 c64:13 c128:11 c128:12}"; WARPS="${2:-16 20 24}"
for cm in $CFG; do
  dt=${cm%%:*}; m=${cm#*:}
  for w in $WARPS; do
    r=$(SV_MIN_WARPS=$w SV_TILE_QUBITS=$m timeout 300 python tools/run_plan.py --dtype $dt 2>&1 | grep "pass ms")
    echo "$dt m=$m warps=$w $r"
  done
done
