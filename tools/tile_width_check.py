"""Per-pass device times of the 30 q supremacy d20 plan at tile widths m (sv_run_opts.tile_qubits)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402
import paper_2106_13995_b200 as P  # noqa: E402

t = W.to_text(W.supremacy(6, 5, 20, seed=0))
for dt in ("c64", "c128"):
    with P.StateVector(30, dt) as sv:
        for m in (0, 12, 13, 14):
            try:
                plan = P.Plan(t, dt, tile_qubits=m, profile=True)
                for _ in range(3):
                    sv.init_zero()
                    sv.apply_plan(plan)
                pt = plan.pass_times()
                print(dt, "m", m, "passes", len(pt), "ms", " ".join(f"{x:.3f}" for x in pt), "total", round(sum(pt), 3),
                      flush=True)
            except Exception as e:
                print(dt, "m", m, "error", str(e)[:200], flush=True)
