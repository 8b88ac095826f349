#!/bin/bash
# pass-pair kernels: parity + bench with and without pairing (SV_PAIR)
O=gpurun_out/${1:-pair}
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_r02.py -q -m gpu -x -rf > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
timeout 300 python bench.py --no-cpu-baseline --no-e2e-cold > $O/bench_pair.log 2>&1
SV_PAIR=0 timeout 300 python bench.py --no-cpu-baseline --no-e2e-cold --no-also > $O/bench_nopair.log 2>&1
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -m gpu -x -rf > $O/fullsize.log 2>&1; echo "exit $?" >> $O/fullsize.log
tail -3 $O/pytest.log $O/fullsize.log
