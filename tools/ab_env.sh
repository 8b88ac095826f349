#!/bin/bash
# A/B per-pass times of the 30 q supremacy plans under environment variants (run under gpurun).
# usage: [REPS=R] [DTYPES="c64 c128"] tools/ab_env.sh OUTDIR "ENV1" "ENV2" ...   ("-" = no extra environment)
# Variants are interleaved R times (power capping drifts over a run); the summary gives the
# median and the minimum total per variant.
O=gpurun_out/$1; shift; mkdir -p $O
for rep in $(seq 1 ${REPS:-2}); do
for v in "$@"; do
  for dt in ${DTYPES:-c64 c128}; do
    r=$(env ${v/#-/} timeout 300 python tools/run_plan.py --dtype $dt 2>&1 | tail -1)
    echo "[$dt] $v: $r" >> $O/ab.txt
  done
done
done
cat $O/ab.txt
python - "$O/ab.txt" <<'PY'
import re, sys, statistics, collections
d = collections.defaultdict(list)
for line in open(sys.argv[1]):
    m = re.match(r"\[(\w+)\] (.*): pass ms: .* total ([\d.]+)", line)
    if m: d[(m.group(1), m.group(2))].append(float(m.group(3)))
print("# summary: dtype variant  median  min  (n)")
for (dt, v), xs in sorted(d.items()):
    print(f"{dt:5s} {v:45s} {statistics.median(xs):8.3f} {min(xs):8.3f}  ({len(xs)})")
PY
