#!/bin/bash
# tile width x pass budget sweep on a bench configuration
ARGS="$1"
for m in 12 13 14; do for b in 110 1000; do
  r=$(SV_TILE_QUBITS=$m SV_PASS_BUDGET=$b python bench.py --steps 5 --warmup 3 --no-cpu-baseline $ARGS 2>/dev/null | tail -1 | python -c "import sys,json; j=json.loads(sys.stdin.read()); print(round(j['ms_per_step'],2), j['config']['passes_per_step'], j['config']['stages_per_step'], round(j['roofline']['frac'],3))")
  echo "[$ARGS] m=$m budget=$b ms/passes/stages/frac: $r"
done; done
