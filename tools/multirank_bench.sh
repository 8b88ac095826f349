#!/bin/bash
# bench.py's N > 1 path with ranks sharing this one GPU (host control plane, CUDA IPC peer
# memory): weak scaling at 2^27 amplitudes per rank, 2 and 4 ranks, fused and copy exchange.
O=gpurun_out/${1:-multirank}
mkdir -p $O
for n in 2 4; do
  python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29500+n)) \
    bench.py --gpus $n --control host --workload weak --qubits 27 --steps 5 --warmup 3 > $O/ranks$n.log 2>&1
  echo "ranks $n: $(grep '^{' $O/ranks$n.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["config"]["n_qubits"], d["config"]["swaps_per_step"], d["config"]["passes_per_step"])')"
done
