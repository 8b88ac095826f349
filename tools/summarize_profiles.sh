#!/bin/bash
# Summaries of a tools/profile_round.sh capture into profiles/ (run here, after gpurun).
R=${1:-r01}
IN=gpurun_out/profile_$R
OUT=profiles
{ echo "# ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none"
  echo "# python bench.py --steps 2 --warmup 3 (30q supremacy d20 c64), B200; per-launch times are serialised/cold"
  python tools/ncu_summary.py launches $IN/launches_bench_c64.csv; } > $OUT/${R}_launches_bench_c64.txt
{ echo "# same, --dtype c128"; python tools/ncu_summary.py launches $IN/launches_bench_c128.csv; } > $OUT/${R}_launches_bench_c128.txt
{ echo "# ncu launch list, 31q 8x7 multiplier c64 (relabel pass + gather pass), two runs"
  python tools/ncu_summary.py launches $IN/launches_mult31.csv; } > $OUT/${R}_launches_mult31.txt
for dt in c64 c128; do
  { echo "# ncu --set full, heaviest tile pass (pass 3) of the 30q supremacy d20 plan, $dt, B200"
    python tools/ncu_summary.py stalls $IN/full_${dt}_raw.csv
    python tools/ncu_summary.py details $IN/full_${dt}_details.csv; } > $OUT/${R}_full_${dt}.txt
  cp $IN/full_${dt}_details.csv $OUT/${R}_full_${dt}_details.csv
done
cp $IN/gpu.txt $OUT/${R}_gpu.txt
