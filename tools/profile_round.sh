#!/bin/bash
# Profiling artefacts of one round (run under gpurun): launch lists of the bench command and
# --set full captures of one mid-circuit tile pass (c64, c128), exported to CSV.
R=${1:-r01}
OUT=gpurun_out/profile_$R
mkdir -p $OUT
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file $OUT/launches_bench_c64.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $OUT/bench_under_ncu.log 2>&1
for dt in c64 c128; do
  ncu --set full --clock-control none --import-source on -k regex:svpass -s 11 -c 1 -o /tmp/full_$dt \
      python tools/run_plan.py --dtype $dt > /dev/null 2>&1
  ncu -i /tmp/full_$dt.ncu-rep --page details --csv > $OUT/full_${dt}_details.csv
  ncu -i /tmp/full_$dt.ncu-rep --page raw --csv > $OUT/full_${dt}_raw.csv
done
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 15 -c 15 \
    --csv --log-file $OUT/launches_mult31.csv python tools/run_plan.py --workload multiplier --qubits 31 > /dev/null 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > $OUT/gpu.txt
