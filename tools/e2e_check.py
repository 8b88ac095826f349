"""e2e step (init + sv_apply_circuit from IR text + 20-qubit marginal to the host) timed by
host wall clock over many steps, 30 q supremacy d20 c64: mean and spread."""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import workloads as W  # noqa: E402
import paper_2106_13995_b200 as P  # noqa: E402

torch.cuda.set_device(0)
text = W.to_text(W.supremacy(6, 5, 20, seed=0))
q = list(range(20))
with P.StateVector(30, "c64") as sv:
    for _ in range(3):
        sv.init_zero()
        sv.apply_circuit(text)
        sv.probabilities(q)
    ts = []
    for _ in range(30):
        t0 = time.perf_counter()
        sv.init_zero()
        sv.apply_circuit(text)
        p = sv.probabilities(q)
        ts.append((time.perf_counter() - t0) * 1e3)
print(f"SV_PINNED={os.environ.get('SV_PINNED', '1')} e2e ms: mean {statistics.mean(ts):.2f} median {statistics.median(ts):.2f} "
      f"min {min(ts):.2f} max {max(ts):.2f}")
