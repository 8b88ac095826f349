#!/bin/bash
# planner knob sweep: ms per circuit for the given bench args, e.g. tools/sweep_budget.sh "--dtype c64"
ARGS="$1"; BUDGETS="${2:-70 110 1000}"
for b in $BUDGETS; do
  r=$(SV_PASS_BUDGET=$b python bench.py --steps 5 --warmup 3 --no-cpu-baseline $ARGS 2>/dev/null | tail -1 | python -c "import sys,json; j=json.loads(sys.stdin.read()); print(round(j['ms_per_step'],2), j['config']['passes_per_step'], j['config']['stages_per_step'], round(j['roofline']['frac'],3))")
  echo "[$ARGS] budget=$b ms/passes/stages/frac: $r"
done
