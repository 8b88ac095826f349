"""BASELINE configs 1 and 2 (small circuits, latency regime): microseconds per circuit and
gates/s on B200, with and without a CUDA graph, next to the oracle.

config 1: 12-qubit supremacy 4x3 grid, 10 cycles, complex128, from |0>.
config 2: 21-qubit multiplier (n = 5), complex128, basis-state inputs (a, b) -> |a,b,ab,0>.
"""
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

torch.cuda.set_device(0)
REPS = 200


def gpu_us(sv, plan, init, reps=REPS):
    stream = torch.cuda.ExternalStream(sv.stream_ptr())
    for _ in range(5):
        init()
        sv.apply_plan(plan)
    sv.sync()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(stream)
    for _ in range(reps):
        init()
        sv.apply_plan(plan)
    e1.record(stream)
    sv.sync()
    wall = (time.perf_counter() - t0) / reps * 1e6
    return e0.elapsed_time(e1) / reps * 1e3, wall


rows = []
c1 = W.supremacy(4, 3, 10, seed=0)
t1 = W.to_text(c1)
for extra in ((4, 4, 10, 16),):  # a 16 q circuit too (3 passes in complex128)
    ce = W.supremacy(extra[0], extra[1], extra[2], seed=0)
    plan = P.Plan(W.to_text(ce), "c128")
    with P.StateVector(extra[3], "c128") as sv:
        dev_us, wall_us = gpu_us(sv, plan, sv.init_zero)
    rows.append({"config": "16q supremacy d10 c128", "gates": W.gate_count(ce), "passes": plan.info()["passes"],
                 "device_us": dev_us, "wall_us": wall_us})
for graph in (False, True):
    plan = P.Plan(t1, "c128", use_graph=graph)
    with P.StateVector(12, "c128") as sv:
        dev_us, wall_us = gpu_us(sv, plan, sv.init_zero)
    rows.append({"config": "1: 12q supremacy d10 c128", "gates": W.gate_count(c1), "graph": graph,
                 "passes": plan.info()["passes"], "device_us": dev_us, "wall_us": wall_us,
                 "gates_per_s_device": W.gate_count(c1) / dev_us * 1e6})
t0 = time.perf_counter()
for _ in range(20):
    oracle.simulate(t1)
rows.append({"config": "1: oracle (fp64, all threads)", "us": (time.perf_counter() - t0) / 20 * 1e6,
             "threads": oracle.max_threads()})

c2 = W.multiplier(5)
t2 = W.to_text(c2)
plan = P.Plan(t2, "c128")
with P.StateVector(c2.n, "c128") as sv:
    x = 19 | (27 << 5)
    dev_us, wall_us = gpu_us(sv, plan, lambda: sv.init_basis(x))
    y = x | ((19 * 27) << 10)
    assert sv.amplitudes(y, 1)[0] == 1
rows.append({"config": "2: 21q multiplier c128, basis input", "gates": W.gate_count(c2),
             "passes": plan.info()["passes"], "device_us": dev_us, "wall_us": wall_us,
             "gates_per_s_device": W.gate_count(c2) / dev_us * 1e6})
psi = np.zeros(1 << c2.n, complex)
psi[x] = 1
t0 = time.perf_counter()
oracle.run(t2, psi)
rows.append({"config": "2: oracle (fp64, all threads)", "us": (time.perf_counter() - t0) * 1e6,
             "threads": oracle.max_threads()})
for r in rows:
    print(json.dumps(r))
