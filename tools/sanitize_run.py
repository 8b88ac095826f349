"""Small run touching every kernel family, for compute-sanitizer (memcheck / racecheck /
synccheck): generated multi-stage tile passes (c64, c128), interpreter and dense-k kernels,
the gather pass with its relabel pass, marginal / norm readout, virtual-sharded exchanges.
Checks results against the oracle so a silent corruption also fails."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import oracle  # noqa: E402
import workloads as W  # noqa: E402
import paper_2106_13995_b200 as P  # noqa: E402


def check(got, ref, tol):
    err = float(np.max(np.abs(got.astype(complex) - ref)))
    assert err <= tol, err


c = W.supremacy(4, 4, 8, seed=1)
t = W.to_text(c)
ref = oracle.simulate(t)
for dt, tol in (("c64", 1e-5), ("c128", 1e-12)):
    for opts in ({}, {"fuse": False}, {"force_kernel": 2}, {"force_kernel": 3}):
        with P.StateVector(16, dt) as sv:
            sv.apply_circuit(t, **opts)
            check(sv.amplitudes(), ref, tol)
            sv.probabilities([0, 5, 15])
            sv.probabilities(list(range(13)))
            sv.norm()
m = W.multiplier(8, 7)
mt = W.to_text(W.concat(W.basis_prep(W.Circuit(31, []), 77 | (99 << 8)), m))
with P.StateVector(31, "c64") as sv:
    sv.apply_circuit(mt)  # relabel pass + gather pass
    y = 77 | (99 << 8) | ((77 * 99) << 15)
    assert sv.amplitudes(y, 1)[0] == 1
rc = W.random_circuit(12, 60, 3, max_k=5, max_controls=2)
rt = W.to_text(rc)
psi0 = W.random_state(12, 3)
with P.StateVector.virtual_sharded(12, 4, "c128") as sv:
    sv.set_amplitudes(psi0)
    sv.apply_circuit(rt)
    check(sv.amplitudes(), oracle.simulate(rt, psi0), 1e-11)
print("sanitize run ok")
