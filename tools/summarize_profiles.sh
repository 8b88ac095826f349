#!/bin/bash
# Summaries of a tools/profile_round.sh capture into profiles/ (run here, after gpurun).
R=${1:-r02}
IN=gpurun_out/profile_$R
OUT=profiles
{ echo "# ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none"
  echo "# python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e-cold (the default bench command: 30q supremacy d20"
  echo "# c64 line, then its c128 and 31q multiplier sub-lines), B200; per-launch times are serialised/cold"
  python tools/ncu_summary.py launches $IN/launches_bench.csv; } > $OUT/${R}_launches_bench.txt
{ echo "# same, c64 line only (--no-also)"; python tools/ncu_summary.py launches $IN/launches_bench_c64.csv; } > $OUT/${R}_launches_bench_c64.txt
{ echo "# same, --dtype c128 --no-also"; python tools/ncu_summary.py launches $IN/launches_bench_c128.csv; } > $OUT/${R}_launches_bench_c128.txt
{ echo "# same, --workload multiplier --qubits 31 (8x7, uniform input synthesised by the relabel pass, then the gather pass)"
  python tools/ncu_summary.py launches $IN/launches_mult31.csv; } > $OUT/${R}_launches_mult31.txt
for spec in c64_supremacy_p0 c64_supremacy_p3 c128_supremacy_p3 c64_multiplier_p1; do
  { echo "# ncu --set full --clock-control none, ${spec}: dtype_workload_pass (tools/run_plan.py, second run), B200"
    python tools/ncu_summary.py stalls $IN/full_${spec}_raw.csv
    python tools/ncu_summary.py details $IN/full_${spec}_details.csv; } > $OUT/${R}_full_${spec}.txt
  cp $IN/full_${spec}_details.csv $OUT/${R}_full_${spec}_details.csv
done
cp $IN/gpu.txt $OUT/${R}_gpu.txt
