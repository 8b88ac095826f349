#!/bin/bash
# Profiling artefacts of one round (run under gpurun): launch lists of the bench commands and
# --set full captures of tile passes of the second run of the plan (c64 pass 0 and pass 3,
# c128 pass 3), exported to CSV; summarised into profiles/ by tools/summarize_profiles.sh.
R=${1:-r01}
OUT=gpurun_out/profile_$R
mkdir -p $OUT
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
ncu --metrics $M --clock-control none --csv --log-file $OUT/launches_bench_c64.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $OUT/bench_under_ncu.log 2>&1
ncu --metrics $M --clock-control none --csv --log-file $OUT/launches_bench_c128.csv \
    python bench.py --dtype c128 --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --metrics $M --clock-control none --csv --log-file $OUT/launches_mult31.csv \
    python bench.py --workload multiplier --qubits 31 --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
# run_plan: 2 runs of the plan, then profiled runs; -s skips to pass p of the second run
for spec in c64:7:p0 c64:10:p3 c128:10:p3; do
  IFS=: read dt skip tag <<< "$spec"
  ncu --set full --clock-control none --import-source on -k regex:svpass -s $skip -c 1 -o /tmp/full_${dt}_$tag \
      python tools/run_plan.py --dtype $dt > /dev/null 2>&1
  ncu -i /tmp/full_${dt}_$tag.ncu-rep --page details --csv > $OUT/full_${dt}_${tag}_details.csv
  ncu -i /tmp/full_${dt}_$tag.ncu-rep --page raw --csv > $OUT/full_${dt}_${tag}_raw.csv
  cp /tmp/full_${dt}_$tag.ncu-rep $OUT/
done
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > $OUT/gpu.txt
