#!/bin/bash
# One GPU verification round (run under gpurun): GPU tests, smoke, the bench lines.
O=gpurun_out/${1:-check}
mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "exit $?" >> $O/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 300 python bench.py > $O/bench_c64.log 2>&1
timeout 300 python bench.py --dtype c128 --no-cpu-baseline > $O/bench_c128.log 2>&1
timeout 300 python bench.py --workload multiplier --qubits 31 --no-cpu-baseline > $O/bench_mult.log 2>&1
timeout 300 python bench.py --impl reference --steps 2 --warmup 3 > $O/bench_reference.log 2>&1
tail -2 $O/pytest_gpu.log
