#!/bin/bash
# late round-2 width sweeps (run under gpurun)
O=gpurun_out/${1:-width}; mkdir -p $O
timeout 1500 python tools/width_sweep.py --family supremacy --min 13 --max 32 > $O/width_sweep_supremacy.jsonl 2>&1
timeout 1500 python tools/width_sweep.py --family multiplier --min 13 --max 32 > $O/width_sweep_multiplier.jsonl 2>&1
tail -3 $O/*.jsonl
