"""the paper's qubit-by-qubit width sweep (Figs. 1-4 methodology)
on B200: for each width, the next larger standard circuit with random qubits removed; GPU
circuit time (c64 and c128, mean of reps, init + passes, plan compiled) and the CPU oracle
(fp64, all host cores) where it is affordable; ratios oracle/GPU.

python tools/width_sweep.py [--family supremacy|multiplier] [--min 13] [--max 30] [--oracle-max 22]
Prints one JSON line per width.
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import workloads as W  # noqa: E402
import paper_2106_13995_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--family", default="supremacy")
ap.add_argument("--min", type=int, default=13)
ap.add_argument("--max", type=int, default=30)
ap.add_argument("--oracle-max", type=int, default=22)
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--depth", type=int, default=20)
a = ap.parse_args()
torch.cuda.set_device(0)

for n in range(a.min, a.max + 1):
    c = W.family_at_width(a.family, n, seed=0, depth=a.depth)
    text = W.to_text(c)
    row = {"family": a.family, "n": n, "gates": W.gate_count(c)}
    for dt in ("c64", "c128"):
        if (16 if dt == "c128" else 8) << n > 120 << 30:
            continue
        plan = P.Plan(text, dt)
        with P.StateVector(n, dt) as sv:
            stream = torch.cuda.ExternalStream(sv.stream_ptr())
            for _ in range(2):  # warm-up (compiles the passes)
                sv.init_uniform()
                sv.apply_plan(plan)
            sv.sync()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(a.reps):
                sv.init_uniform()  # equal-superposition input, as the paper
                st = sv.apply_plan(plan)
            e1.record(stream)
            sv.sync()
            ms = e0.elapsed_time(e1) / a.reps
        row[f"gpu_{dt}_ms"] = ms
        row[f"passes_{dt}"] = st["passes"]
    if n <= a.oracle_max:
        psi = oracle.uniform_state(n)
        t0 = time.perf_counter()
        oracle.run(text, psi)
        row["oracle_ms"] = (time.perf_counter() - t0) * 1e3
        row["oracle_threads"] = oracle.max_threads()
        row["speedup_c128"] = row["oracle_ms"] / row["gpu_c128_ms"]
    print(json.dumps(row), flush=True)
