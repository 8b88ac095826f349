mkdir -p gpurun_out/r3
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r3/pytest_gpu.log 2>&1; echo "exit $?" >> gpurun_out/r3/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r3/smoke.log 2>&1
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/r3/bench_c64.log 2>&1
timeout 300 python bench.py --dtype c128 --no-cpu-baseline > gpurun_out/r3/bench_c128.log 2>&1
SV_MERGE1Q=0 timeout 300 python bench.py --no-cpu-baseline > gpurun_out/r3/bench_c64_nomerge.log 2>&1
timeout 300 python tools/run_plan.py --dtype c64 > gpurun_out/r3/passes_c64.log 2>&1
timeout 300 python tools/run_plan.py --dtype c128 > gpurun_out/r3/passes_c128.log 2>&1
tail -2 gpurun_out/r3/pytest_gpu.log
