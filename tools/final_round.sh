#!/bin/bash
# End-of-round verification (run under gpurun): GPU tests, smoke, bench lines (default,
# reference arm), and the launch list of the default bench command.
O=gpurun_out/${1:-final}
mkdir -p $O
timeout 2000 python -m pytest tests -q -m gpu -rf > $O/pytest_gpu.log 2>&1; echo "exit $?" >> $O/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 600 python bench.py > $O/bench.log 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > $O/bench_reference.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $O/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e-cold > /dev/null 2>&1
tail -3 $O/pytest_gpu.log; tail -1 $O/smoke.log
