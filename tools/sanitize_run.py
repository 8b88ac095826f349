"""Small run touching every kernel family, for compute-sanitizer (memcheck / racecheck /
synccheck): generated multi-stage tile passes (c64, c128), interpreter and dense-k kernels,
the gather pass with its relabel pass, marginal / norm readout, virtual-sharded exchanges.
Round-1 additions: fused / peer-copy exchange, dense-k single gates, deferred uniform input.
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
# this round's additions: fused peer-memory exchange (remote-store pass variants) and the
# peer-copy kernel after interpreter passes, c64 and c128, P = 2 and 8
for dt, tol in (("c64", 1e-5), ("c128", 1e-12)):
    for world in (2, 8):
        for opts in ({}, {"fuse": False}):
            with P.StateVector.virtual_sharded(16, world, dt) as sv:
                st = sv.apply_circuit(t, **opts)
                assert st["swaps"] >= 1
                check(sv.amplitudes(), ref, tol)
# single gates through the dense-k kernels (k = 1..3, with/without controls, qubit 0 free or not)
h = 2 ** -0.5
u2 = np.linalg.qr(np.random.default_rng(1).normal(size=(4, 4)) + 0j)[0]
u3 = np.linalg.qr(np.random.default_rng(2).normal(size=(8, 8)) + 0j)[0]
for dt, tol in (("c64", 1e-5), ("c128", 1e-12)):
    psi0 = W.random_state(14, 5)
    ref2 = psi0.copy()
    with P.StateVector(14, dt) as sv:
        sv.set_amplitudes(psi0)
        for U, tg, ct in ((np.array([[h, h], [h, -h]]), [0], []), (np.array([[h, h], [h, -h]]), [9], [0]),
                          (u2, [3, 11], []), (u2, [1, 0], [13]), (u3, [2, 7, 12], []), (u3, [4, 5, 6], [0, 1])):
            sv.apply_gate(U, tg, ct)
            ref2 = oracle.apply_gate(ref2, U, tg, ct)
        check(sv.amplitudes(), ref2, tol if dt == "c128" else 1e-5)
# deferred uniform input synthesised by the first pass; merged unit-class runs
for dt, tol in (("c64", 1e-5), ("c128", 1e-12)):
    with P.StateVector(16, dt) as sv:
        sv.init_uniform()
        sv.apply_circuit(t)
        check(sv.amplitudes(), oracle.simulate(t, np.full(1 << 16, 2.0 ** -8, complex)), tol)
print("sanitize run ok")

# Round-2 additions: borrowed buffer canonicalised after a relabelling plan (sv_wrap),
# sv_device_ptr canonicalisation, dense-k with many controls (bit-insertion table), and the
# pass-pair kernels (SV_PAIR=1 is read once per process: enabled here through the env var
# set by the caller, else skipped).
import torch  # noqa: E402

c = W.supremacy(4, 4, 10, seed=3)
t = W.to_text(c)
ref = oracle.simulate(t)
for dt, tol in (("c64", 1e-5), ("c128", 1e-12)):
    buf = torch.zeros(1 << 16, dtype=torch.complex64 if dt == "c64" else torch.complex128, device="cuda")
    buf[0] = 1
    with P.StateVector.wrap(buf, 16) as sv:
        sv.apply_circuit(t)
        sv.sync()
        check(buf.cpu().numpy(), ref, tol)
    with P.StateVector(16, dt) as sv:
        sv.apply_circuit(t)
        sv.device_ptr()
        check(sv.amplitudes(), ref, tol)
n = 16
psi0 = W.random_state(n, 5)
X = np.array([[0, 1], [1, 0]], complex)
ctl = list(range(1, 15))
want = psi0.copy()
idx = np.flatnonzero([all((i >> q) & 1 for q in ctl) for i in range(1 << n)])
want[idx] = oracle.apply_gate(np.ascontiguousarray(psi0[idx]), X, [0])
with P.StateVector(n, "c128") as sv:
    sv.set_amplitudes(psi0)
    sv.apply_gate(X, [0], ctl)
    check(sv.amplitudes(), want, 1e-14)
if os.environ.get("SV_PAIR") == "1":
    c = W.supremacy(5, 4, 14, seed=2)
    t = W.to_text(c)
    ref = oracle.simulate(t)
    with P.StateVector(20, "c64") as sv:
        sv.apply_circuit(t)
        check(sv.amplitudes(), ref, 1e-5)
print("sanitize run (round-2 paths) ok")

# small-state schedule in one kernel (grid barrier between passes), all input variants
c = W.supremacy(4, 3, 10, seed=0)
t = W.to_text(c)
ref = oracle.simulate(t)
for dt, tol in (("c64", 1e-5), ("c128", 1e-12)):
    with P.StateVector(12, dt) as sv:
        for _ in range(3):
            sv.init_zero()
            sv.apply_circuit(t)
            check(sv.amplitudes(), ref, tol)
        sv.init_uniform()
        sv.apply_circuit(t)
        check(sv.amplitudes(), oracle.simulate(t, np.full(1 << 12, 2.0 ** -6, complex)), tol)
print("sanitize run (small-state schedule) ok")
