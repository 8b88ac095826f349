#!/bin/bash
# Bench lines of the round (run under gpurun): default line (config 3 c64 + also c128 / config 4,
# e2e_cold, cpu_baseline), reference arm, strong33 at N = 1, width sweeps.
O=gpurun_out/${1:-bench}
mkdir -p $O
timeout 600 python bench.py > $O/bench.log 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > $O/bench_reference.log 2>&1
timeout 600 python bench.py --workload strong33 --steps 5 --no-cpu-baseline --no-e2e-cold > $O/bench_strong33.log 2>&1
timeout 900 python tools/width_sweep.py --family supremacy --min 13 --max 32 > $O/width_sweep_supremacy.jsonl 2>&1
timeout 900 python tools/width_sweep.py --family multiplier --min 13 --max 32 > $O/width_sweep_multiplier.jsonl 2>&1
tail -c 600 $O/bench.log
