#!/bin/bash
# Per-launch device time of every pass of the second run of a plan under ncu with locked base
# clocks (--clock-control ${CLOCK:-base}: a fair A/B when power capping moves the clocks), per env variant.
# usage: DTYPE=c128 tools/ncu_ab.sh OUT "ENV1" "ENV2" ...
O=gpurun_out/$1; shift; mkdir -p $O
for v in "$@"; do
  env ${v/#-/} timeout 600 ncu --metrics gpu__time_duration.sum --clock-control ${CLOCK:-base} -k regex:svpass --csv \
      python tools/run_plan.py --dtype ${DTYPE:-c128} --reps 2 2>/dev/null | grep svpass > $O/raw_$(echo "$v" | tr ' =/' '___').csv
  python - "$O/raw_$(echo "$v" | tr ' =/' '___').csv" "$v" <<'PY'
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
t = [float(r[-1].replace(",", "")) / 1e6 for r in rows if r and r[-3] == "gpu__time_duration.sum"]
n = len(t) // 5 if len(t) >= 10 else len(t)
print(f"{sys.argv[2]:35s} launches {len(t)}: " + " ".join(f"{x:.3f}" for x in t[:16]))
PY
done
