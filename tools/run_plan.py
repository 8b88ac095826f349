"""Profiling driver: run one circuit plan `reps` times on a fresh state (for ncu captures).

python tools/run_plan.py [--workload supremacy|multiplier] [--dtype c64] [--qubits 30] [--reps 2]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import workloads as W  # noqa: E402
import paper_2106_13995_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="supremacy")
ap.add_argument("--dtype", default="c64")
ap.add_argument("--qubits", type=int, default=30)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--fuse", type=int, default=1)
a = ap.parse_args()
if a.workload == "supremacy":
    c = W.supremacy(6, 5, 20, 0) if a.qubits == 30 else W.supremacy((a.qubits + 4) // 5, 5, 20, 0, n=a.qubits)
elif a.workload == "qft":
    c = W.qft(a.qubits)
else:
    c = W.multiplier(8, 7)
plan = P.Plan(W.to_text(c), a.dtype, fuse=bool(a.fuse))
with P.StateVector(c.n, a.dtype) as sv:
    for _ in range(a.reps):
        sv.init_zero()
        st = sv.apply_plan(plan)
    sv.sync()
print(st, plan.info())

# per-pass device times of a back-to-back run (CUDA events between launches); RUN_PLAN_COOL=s
# idles s seconds first (A/B runs under power capping: every variant starts from the same state)
if os.environ.get("RUN_PLAN_COOL"):
    import time
    time.sleep(float(os.environ["RUN_PLAN_COOL"]))
pplan = P.Plan(W.to_text(c), a.dtype, fuse=bool(a.fuse), profile=True)
with P.StateVector(c.n, a.dtype) as sv:
    for _ in range(3):
        sv.init_zero()
        sv.apply_plan(pplan)
    t = pplan.pass_times()
    print("pass ms:", " ".join(f"{x:.3f}" for x in t), " total", round(sum(t), 3))
