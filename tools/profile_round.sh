#!/bin/bash
# Profiling artefacts of one round (run under gpurun): the launch list of the default bench
# command (config 3 c64 line + its c128 / config-4 sub-lines) and per-workload lists, and
# --set full captures of tile passes of the second run of the plan (c64 pass 0 and pass 3,
# c128 pass 3) and of the config-4 gather pass; summarised into profiles/ by
# tools/summarize_profiles.sh.
R=${1:-r02}
OUT=gpurun_out/profile_$R
mkdir -p $OUT
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
ncu --metrics $M --clock-control none --csv --log-file $OUT/launches_bench.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e-cold > $OUT/bench_under_ncu.log 2>&1
ncu --metrics $M --clock-control none --csv --log-file $OUT/launches_bench_c64.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e-cold --no-also > /dev/null 2>&1
ncu --metrics $M --clock-control none --csv --log-file $OUT/launches_bench_c128.csv \
    python bench.py --dtype c128 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e-cold --no-also > /dev/null 2>&1
ncu --metrics $M --clock-control none --csv --log-file $OUT/launches_mult31.csv \
    python bench.py --workload multiplier --qubits 31 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e-cold > /dev/null 2>&1
# run_plan: 2 runs of the plan, then profiled runs; -s skips to pass p of the second run
for spec in c64:supremacy:7:p0 c64:supremacy:10:p3 c128:supremacy:10:p3 c64:multiplier:3:p1; do
  IFS=: read dt wl skip tag <<< "$spec"
  ncu --set full --clock-control none --import-source on -k regex:svpass -s $skip -c 1 -o /tmp/full_${dt}_${wl}_$tag \
      python tools/run_plan.py --dtype $dt --workload $wl $( [ $wl = multiplier ] && echo --qubits 31 ) > /dev/null 2>&1
  ncu -i /tmp/full_${dt}_${wl}_$tag.ncu-rep --page details --csv > $OUT/full_${dt}_${wl}_${tag}_details.csv
  ncu -i /tmp/full_${dt}_${wl}_$tag.ncu-rep --page raw --csv > $OUT/full_${dt}_${wl}_${tag}_raw.csv
  cp /tmp/full_${dt}_${wl}_$tag.ncu-rep $OUT/
done
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > $OUT/gpu.txt
