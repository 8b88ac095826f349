"""Latency of small supremacy circuits (12 / 14 / 16 / 18 q, depth 10) per dtype: device us per
circuit (mean of 200 back-to-back runs from |0>), plan shape.  python tools/small_lat.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import workloads as W  # noqa: E402
import paper_2106_13995_b200 as P  # noqa: E402

torch.cuda.set_device(0)
# default: 12 / 14 / 16 / 18 q; --medium: 18 / 20 / 22 / 24 q
GRIDS = ((6, 3), (5, 4), (11, 2), (6, 4)) if "--medium" in sys.argv else ((4, 3), (7, 2), (4, 4), (6, 3))
for dt in ("c128", "c64"):
    for rows, cols in GRIDS:
        c = W.supremacy(rows, cols, 10, seed=0)
        plan = P.Plan(W.to_text(c), dt)
        with P.StateVector(c.n, dt) as sv:
            st = torch.cuda.ExternalStream(sv.stream_ptr())
            for _ in range(5):
                sv.init_zero()
                sv.apply_plan(plan)
            sv.sync()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for _ in range(200):
                sv.init_zero()
                sv.apply_plan(plan)
            e1.record(st)
            sv.sync()
            print(json.dumps({"dtype": dt, "n": c.n, "gates": W.gate_count(c), "passes": plan.info()["passes"],
                              "device_us": round(e0.elapsed_time(e1) / 200 * 1e3, 2), "rb": os.environ.get("SV_RB", "default")}))
