#!/bin/bash
# Quick GPU check after a generator change (run under gpurun): parity tests except the
# full-size ones, then the bench line and per-pass times.  Output in gpurun_out/$1.
O=gpurun_out/${1:-quick}
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_r02.py -q -m gpu -x -rf > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
timeout 300 python tools/run_plan.py > $O/plan_c64.log 2>&1
timeout 300 python tools/run_plan.py --dtype c128 > $O/plan_c128.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-e2e-cold > $O/bench.log 2>&1
tail -2 $O/pytest.log; tail -1 $O/plan_c64.log; tail -1 $O/plan_c128.log
