"""Fused vs copy exchange on one GPU, through virtual sharding.

An n-qubit supremacy circuit split into P virtual shards of one allocation runs the sharded
planner; its global<->local swaps are either fused into the
preceding pass (stores into the second buffer pair at the swapped positions; exchange=0) or
done after it as in-place chunk swaps (device copies through a staging chunk; exchange=1 --
the single-GPU stand-in for the NCCL send/recv path).  Device time per circuit with CUDA
events on the state's stream, after warm-up.  On one GPU the "peer" stores are local HBM
stores, so this measures the HBM round trip the fusion saves, not NVLink.

python tools/exchange_bench.py [--qubits 30] [--world 2] [--dtype c64] [--reps 5]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import workloads as W  # noqa: E402
import paper_2106_13995_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--qubits", type=int, default=30)
ap.add_argument("--world", type=int, default=2)
ap.add_argument("--dtype", default="c64")
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
n = a.qubits
c = W.supremacy((n + 4) // 5, 5, 20, seed=0, n=n) if n != 30 else W.supremacy(6, 5, 20, seed=0)
text = W.to_text(c)
out = {"qubits": n, "world": a.world, "dtype": a.dtype, "gates": len(c.gates)}
for mode, name in ((0, "fused"), (1, "copy")):
    plan = P.Plan(text, a.dtype, exchange=mode)
    with P.StateVector.virtual_sharded(n, a.world, a.dtype) as sv:
        stream = torch.cuda.ExternalStream(sv.stream_ptr())
        for _ in range(2):
            sv.init_zero()
            st = sv.apply_plan(plan)
        sv.sync()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.reps)]
        for e0, e1 in ev:
            sv.init_zero()
            e0.record(stream)
            st = sv.apply_plan(plan)
            e1.record(stream)
        sv.sync()
        ms = sorted(e0.elapsed_time(e1) for e0, e1 in ev)
        out[name] = {"ms_median": ms[len(ms) // 2], "ms_min": ms[0], "swaps": st["swaps"], "passes": st["passes"],
                     "launches": st["launches"]}
    plan.close()
out["saved_ms"] = out["copy"]["ms_median"] - out["fused"]["ms_median"]
print(json.dumps(out))
