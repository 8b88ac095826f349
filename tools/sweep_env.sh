#!/bin/bash
# Environment-knob sweep: total device ms of the passes of one plan per setting.
# usage: tools/sweep_env.sh "--dtype c64" "SV_TPC=1 SV_TILE_QUBITS=12" "SV_TPC=2 SV_TILE_QUBITS=12" ...
ARGS="$1"; shift
for setting in "$@"; do
  r=$(env $setting timeout 300 python tools/run_plan.py $ARGS 2>&1 | grep "pass ms")
  echo "[$ARGS] $setting: $r"
done
