"""compute-sanitizer target for the round-2 kernels only (small-state schedule, wrap
canonicalisation, many-control dense-k): quick to run under racecheck."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
import workloads as W  # noqa: E402
import paper_2106_13995_b200 as P  # noqa: E402

c = W.supremacy(4, 3, 10, seed=0)
t = W.to_text(c)
ref = oracle.simulate(t)
for dt, tol in (("c64", 1e-5), ("c128", 1e-12)):
    with P.StateVector(12, dt) as sv:
        for _ in range(3):
            sv.init_zero()
            sv.apply_circuit(t)
            assert float(np.max(np.abs(sv.amplitudes() - ref))) <= tol
print("small-state schedule ok")
