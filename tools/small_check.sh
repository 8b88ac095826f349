#!/bin/bash
O=gpurun_out/${1:-small}
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_r02.py -q -m gpu -x -rf > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
for v in 1 0 1 0; do echo "== SV_SMALL_FUSE=$v" >> $O/small.txt; SV_SMALL_FUSE=$v timeout 300 python tools/small_circuits.py >> $O/small.txt 2>&1; done
tail -3 $O/pytest.log; cat $O/small.txt
