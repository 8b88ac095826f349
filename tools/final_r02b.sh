#!/bin/bash
# Late round-2 measurement set (run under gpurun): bench line (default), reference arm, launch
# list of the default bench command, --set full captures of the key passes.
O=gpurun_out/${1:-final_b}
mkdir -p $O
timeout 600 python bench.py > $O/bench.log 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > $O/bench_reference.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $O/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e-cold > /dev/null 2>&1
bash tools/profile_late.sh ${1:-final_b}_prof
tail -c 400 $O/bench.log
