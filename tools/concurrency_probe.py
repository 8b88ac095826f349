"""Probe: do two pass sequences on independent states overlap their FP-heavy and HBM-heavy
passes when run concurrently on two streams (B started one pass later than A)?

python tools/concurrency_probe.py [--qubits 29] [--dtype c64] [--delay-ms 3]
Prints the device time of A alone, and of A and B together (staggered), both after warm-up.
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
ap.add_argument("--qubits", type=int, default=29)
ap.add_argument("--dtype", default="c64")
ap.add_argument("--delay-ms", type=float, default=3.0)
a = ap.parse_args()
n = a.qubits
c = W.supremacy(6, 5, 20, seed=0, n=n)
text = W.to_text(c)
plan = P.Plan(text, a.dtype)
sA = torch.cuda.Stream()
sB = torch.cuda.Stream()
A = P.StateVector(n, a.dtype, stream=sA.cuda_stream)
B = P.StateVector(n, a.dtype, stream=sB.cuda_stream)
for _ in range(2):
    A.init_zero(); A.apply_plan(plan)
    B.init_zero(); B.apply_plan(plan)
torch.cuda.synchronize()


def timed(fn):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    fn()
    torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


def alone():
    A.init_zero(); A.apply_plan(plan)


cycles = int(a.delay_ms * 1e-3 * 1.9e9)


def both(delay=True):
    e = torch.cuda.Event()
    e.record()
    sA.wait_event(e)
    sB.wait_event(e)
    if delay:
        with torch.cuda.stream(sB):
            torch.cuda._sleep(cycles)
    A.init_zero(); A.apply_plan(plan)
    B.init_zero(); B.apply_plan(plan)


def sleep_only():
    with torch.cuda.stream(sB):
        torch.cuda._sleep(cycles)


res = {"qubits": n, "dtype": a.dtype, "passes": plan.info()["passes"]}
res["alone_ms"] = min(timed(alone) for _ in range(3))
res["sleep_ms"] = min(timed(sleep_only) for _ in range(3))
res["both_staggered_ms"] = min(timed(both) for _ in range(3))
res["both_unstaggered_ms"] = min(timed(lambda: both(False)) for _ in range(3))
# serial execution would take 2 x alone; perfect overlap about alone + the stagger
res["serial_ms"] = 2 * res["alone_ms"]
print(json.dumps(res))
