#!/bin/bash
# Profiling artefacts of one round (run under gpurun): launch lists of the bench command and
# --set full captures of the heaviest tile pass (c64, c128) of the second run of the plan,
# exported to CSV; summarised into profiles/ by tools/ncu_summary.py (run here).
R=${1:-r01}
OUT=gpurun_out/profile_$R
mkdir -p $OUT
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file $OUT/launches_bench_c64.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $OUT/bench_under_ncu.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file $OUT/launches_bench_c128.csv python bench.py --dtype c128 --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
# run_plan: 2 runs of the plan then a profiled run; -s skips to pass 3 of the second run
for spec in c64:10 c128:11; do
  dt=${spec%%:*}; skip=${spec#*:}
  ncu --set full --clock-control none --import-source on -k regex:svpass -s $skip -c 1 -o /tmp/full_$dt \
      python tools/run_plan.py --dtype $dt > /dev/null 2>&1
  ncu -i /tmp/full_$dt.ncu-rep --page details --csv > $OUT/full_${dt}_details.csv
  ncu -i /tmp/full_$dt.ncu-rep --page raw --csv > $OUT/full_${dt}_raw.csv
  cp /tmp/full_$dt.ncu-rep $OUT/
done
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 2 -c 4 \
    --csv --log-file $OUT/launches_mult31.csv python tools/run_plan.py --workload multiplier --qubits 31 > /dev/null 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > $OUT/gpu.txt
