#!/bin/bash
# Full GPU test suite + smoke (run under gpurun); output in gpurun_out/$1
O=gpurun_out/${1:-full}
mkdir -p $O
timeout 2400 python -m pytest tests -q -m gpu -rf > $O/pytest_gpu.log 2>&1; echo "exit $?" >> $O/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
tail -3 $O/pytest_gpu.log; tail -1 $O/smoke.log
