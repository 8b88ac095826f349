"""Parity cases added in round 2 (VERDICT r01 "what's weak" 1, 3, 6, 7).

* Configs 2 and 4 at their exact plans (relabel pass + bit-sliced gather pass) on seeded
  random inputs: psi_out[f(i)] == psi_in[i] at EVERY index (SURVEY 8(c) comparison step 5),
  f from the oracle's classical map; 21 q also against oracle.simulate bit for bit.
* Removal-derived circuits of both families vs the oracle.
* Borrowed buffers (sv_wrap) hold the state in index order after a relabelling plan.
* Gates with more controls than the old dense-parameter block held.
* Near-unit custom gates keep their deviation from the unit class (reading "unit-class snap").
"""

import numpy as np
import pytest

import oracle
import workloads as W
from tests.parity import assert_close

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_2106_13995_b200 as P
    return P


class _DevView:
    """Zero-copy torch view of a device buffer (test harness only: comparisons on the GPU)."""

    def __init__(self, ptr, n, typestr):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False), "version": 3}


def _state_tensor(torch, sv, dtype):
    ptr, n = sv.device_ptr()  # canonical layout (logical index order), queued on sv's stream
    sv.sync()
    return torch.as_tensor(_DevView(ptr, n, "<c8" if dtype == "c64" else "<c16"), device="cuda")


# ------------------------------------------------------------------ configs 2 / 4, exact plans
def test_config2_exact_plan_random_state_bit_exact(P):
    """Config 2 (21 q multiplier, c128): the plan sv_apply_circuit compiles (relabel + gather)
    on a seeded random normalised state, against oracle.simulate at every amplitude (==)."""
    c = W.multiplier(5)
    text = W.to_text(c)
    plan = P.Plan(text, "c128")
    kinds = [("permutation pass" in plan.source(i)) for i in range(plan.info()["passes"])]
    assert kinds[-1] and plan.qubit_map() != list(range(c.n))  # relabel + gather, as timed
    psi0 = W.random_state(c.n, 2021)
    with P.StateVector(c.n, "c128") as sv:
        sv.set_amplitudes(psi0)
        sv.apply_plan(plan)
        got = sv.amplitudes()
    ref = oracle.simulate(text, psi0)
    assert np.array_equal(got, ref)
    f = oracle.classical_map_range(text, 0, 1 << c.n).astype(np.int64)
    assert np.array_equal(got[f], psi0)


def test_config4_exact_plan_random_state_every_index(P):
    """Config 4 at full width (31 q 8x7 multiplier, c64), the plan bench.py times (relabel +
    gather), on a seeded random input: psi_out[f(i)] == psi_in[i] bit for bit for all 2^31 i,
    f from the oracle's bit-sliced classical map (chunked)."""
    import torch
    c = W.multiplier(8, 7)
    text = W.to_text(c)
    n = c.n
    plan = P.Plan(text, "c64")
    info = plan.info()
    assert info["passes"] == 2 and "permutation pass" in plan.source(1)
    N = 1 << n
    gen = torch.Generator(device="cuda")
    gen.manual_seed(31)
    psi_in = torch.randn(N, dtype=torch.complex64, device="cuda", generator=gen)
    with P.StateVector(n, "c64") as sv:
        _state_tensor(torch, sv, "c64").copy_(psi_in)
        torch.cuda.synchronize()
        sv.apply_plan(plan)
        out = _state_tensor(torch, sv, "c64")  # re-queried: the gather pass swaps buffers
        torch.cuda.synchronize()
        a_in = torch.view_as_real(psi_in).view(torch.int64)  # bitwise comparison
        a_out = torch.view_as_real(out).view(torch.int64)
        chunk = 1 << 26
        f = np.empty(chunk, dtype=np.uint64)
        bad = 0
        for first in range(0, N, chunk):
            oracle.classical_map_range(text, first, chunk, f)
            idx = torch.from_numpy(f.view(np.int64)).to("cuda", non_blocking=False)
            bad += int((a_out[idx] != a_in[first:first + chunk]).sum())
        assert bad == 0


# ------------------------------------------------------------------ f3: removal-derived circuits
@pytest.mark.parametrize("n", [14, 18, 19])
def test_removal_derived_multiplier_exact(P, n):
    """widths between 4k+1 and 4(k+1)+1 come from the larger multiplier with random
    qubits removed.  Still a classical reversible circuit: exact on a random input."""
    c = W.family_at_width("multiplier", n, seed=n)
    assert c.n == n and c.meta.get("removed")
    text = W.to_text(c)
    psi0 = W.random_state(n, 300 + n)
    for dtype in ("c128", "c64"):
        x = psi0 if dtype == "c128" else W.round_to_c64(psi0)
        with P.StateVector(n, dtype) as sv:
            sv.set_amplitudes(x)
            sv.apply_circuit(text)
            got = sv.amplitudes()
        assert np.array_equal(got.astype(np.complex128), oracle.simulate(text, x.astype(np.complex128)))


@pytest.mark.parametrize("n", [19, 23, 26])
@pytest.mark.parametrize("dtype", ["c128", "c64"])
def test_removal_derived_supremacy(P, n, dtype):
    """a 19-qubit supremacy circuit is the 20-qubit (5x4) one minus a random qubit."""
    c = W.family_at_width("supremacy", n, seed=5, depth=14)
    assert c.n == n
    text = W.to_text(c)
    with P.StateVector(n, dtype) as sv:
        sv.apply_circuit(text)
        got = sv.amplitudes()
    assert_close(got, oracle.simulate(text), dtype, W.gate_count(c))


# ------------------------------------------------------------------ boundary: borrowed buffers
@pytest.mark.parametrize("dtype", ["c64", "c128"])
def test_wrap_supremacy_tensor_in_index_order(P, dtype):
    """sv_wrap + a relabelling plan (20 q supremacy): the caller's tensor, read directly after
    a sync, holds the state in logical index order."""
    import torch
    n = 20
    c = W.supremacy(5, 4, 16, seed=0)
    text = W.to_text(c)
    assert P.Plan(text, dtype).qubit_map() != list(range(n))  # the plan ends relabelled
    t = torch.zeros(1 << n, dtype=torch.complex64 if dtype == "c64" else torch.complex128, device="cuda")
    t[0] = 1
    with P.StateVector.wrap(t, n) as sv:
        sv.apply_circuit(text)
        assert sv.qubit_map() == list(range(n))
        sv.sync()
        got = t.cpu().numpy()
    assert_close(got, oracle.simulate(text), dtype, W.gate_count(c))


def test_device_ptr_is_canonical(P):
    """An owned state left relabelled by its plan: sv_device_ptr hands out index order."""
    import torch
    n = 20
    text = W.to_text(W.supremacy(5, 4, 16, seed=1))
    with P.StateVector(n, "c128") as sv:
        sv.apply_circuit(text)
        assert sv.qubit_map() != list(range(n))
        view = _state_tensor(torch, sv, "c128")
        torch.cuda.synchronize()
        assert sv.qubit_map() == list(range(n))
        got = view.cpu().numpy()
    assert_close(got, oracle.simulate(text), "c128", 1000)


# ------------------------------------------------------------------ many controls (dense params)
def _controlled_ref(psi, n, U, targets, controls):
    """Reference for a gate with many controls: the oracle applies U (uncontrolled) to the
    sub-state where every control bit is 1 (the gate acts as U there and as the
    identity elsewhere); the oracle's own controlled form is limited to 5 qubits in total."""
    rest = [q for q in range(n) if q not in controls]
    idx = np.zeros(1 << len(rest), dtype=np.int64)
    for j, q in enumerate(rest):
        idx |= ((np.arange(1 << len(rest)) >> j) & 1) << q
    for q in controls:
        idx |= 1 << q
    out = psi.copy()
    sub = np.ascontiguousarray(psi[idx])
    out[idx] = oracle.apply_gate(sub, U, [rest.index(t) for t in targets])
    return out


@pytest.mark.parametrize("nctl", [12, 14, 17])
@pytest.mark.parametrize("dtype", ["c128", "c64"])
def test_apply_gate_many_controls(P, nctl, dtype):
    """sv_apply_gate with k <= 3 takes the dense-k kernel; controls + targets beyond 12 used
    to overflow its bit-insertion table."""
    n = 20
    psi0 = W.random_state(n, nctl)
    psi0 = W.round_to_c64(psi0) if dtype == "c64" else psi0
    ctl = list(range(1, nctl + 1))
    X = np.array([[0, 1], [1, 0]], complex)
    U2 = W.random_unitary(2, np.random.default_rng(7))
    ref = _controlled_ref(psi0.astype(complex), n, X, [0], ctl)
    ref = _controlled_ref(ref, n, U2, [19, 0], ctl[:-1])
    with P.StateVector(n, dtype) as sv:
        sv.set_amplitudes(psi0)
        sv.apply_gate(X, [0], ctl)
        sv.apply_gate(U2, [19, 0], ctl[:-1])
        got = sv.amplitudes()
    assert_close(got, ref, dtype, 2)


# ------------------------------------------------------------------ unit-class snap
def test_near_unit_custom_gates_keep_their_deviation(P):
    """2000 custom rotations R(pi/4 + d), d = 1e-13, on one qubit: each is within 1e-13 of the
    unit-class matrix R(pi/4) ~ H-like, which the planner must NOT substitute (the old 1e-12
    snap did, accumulating 2000 d = 2e-10 of rotation).  Against the oracle at 1e-12 (c128)."""
    n = 4
    th = np.pi / 4 + 1e-13
    R = np.array([[np.cos(th), -np.sin(th)], [np.sin(th), np.cos(th)]])
    lines = [f"qubits: {n}", "H 0; H 2"]
    nums = ",".join(f"{float(v)!r},0.0" for v in R.reshape(-1))
    for i in range(2000):
        lines.append(f"U 1 : {nums}")
        if i % 100 == 99:
            lines.append("CZ 1,2")
    text = "\n".join(lines) + "\n"
    with P.StateVector(n, "c128") as sv:
        sv.apply_circuit(text)
        got = sv.amplitudes()
    ref = oracle.simulate(text)
    assert np.max(np.abs(got - ref)) <= 1e-12


# ------------------------------------------------------------------ wide dense blocks at size
@pytest.mark.parametrize("dtype", ["c128", "c64"])
@pytest.mark.parametrize("mode", [{}, {"force_kernel": 2}])
def test_wide_dense_blocks_21q(P, dtype, mode):
    """k = 4, 5 dense / controlled blocks at 21 q (dense-k kernels with many blocks and a
    grid-stride tail; fused: OP_U4 in registers, k = 5 as dense passes) against the oracle."""
    n = 21
    c = W.random_circuit(n, 40, 2121, kinds=["U", "CU", "Udiag", "H", "CZ"], max_k=5, max_controls=2)
    text = W.to_text(c)
    psi0 = W.random_state(n, 21)
    psi0 = W.round_to_c64(psi0) if dtype == "c64" else psi0
    with P.StateVector(n, dtype) as sv:
        sv.set_amplitudes(psi0)
        sv.apply_circuit(text, **mode)
        got = sv.amplitudes()
    assert_close(got, oracle.simulate(text, psi0.astype(complex)), dtype, W.gate_count(c))


@pytest.mark.parametrize("dtype", ["c128", "c64"])
def test_apply_gate_wide_blocks_with_controls(P, dtype):
    """sv_apply_gate with k = 4, 5 (dense_kw) with and without controls, targets unsorted and
    including qubit 0."""
    n = 18
    psi0 = W.random_state(n, 4)
    psi0 = W.round_to_c64(psi0) if dtype == "c64" else psi0
    ref = psi0.astype(complex)
    rng = np.random.default_rng(5)
    with P.StateVector(n, dtype) as sv:
        sv.set_amplitudes(psi0)
        for k, tg, ct in ((4, [7, 0, 13, 2], []), (5, [17, 3, 0, 9, 11], []), (4, [1, 5, 6, 16], [0]),
                          (5, [2, 4, 8, 10, 12], [15, 1])):
            U = W.random_unitary(k, rng)
            sv.apply_gate(U, tg, ct)
            ref = oracle.apply_gate(ref, U, tg, ct)
        got = sv.amplitudes()
    assert_close(got, ref, dtype, 4)


def test_plan_cache_concurrent_threads(P):
    """sv_apply_circuit's process-wide plan cache under concurrency: 4 host
    threads, each with its own state, apply 24 distinct circuits (more than the 16 cached
    plans, so entries are evicted while other threads use them) and one shared circuit;
    every result matches the oracle."""
    import threading
    n = 10
    texts = [W.to_text(W.random_circuit(n, 30, 900 + i, max_k=3)) for i in range(24)]
    shared = W.to_text(W.supremacy(5, 2, 8, seed=9))
    refs = [oracle.simulate(t) for t in texts]
    ref_shared = oracle.simulate(shared)
    errors = []

    def work(tid):
        try:
            with P.StateVector(n, "c128") as sv:
                for r in range(3):
                    for i in range(tid, len(texts), 4):
                        sv.init_zero()
                        sv.apply_circuit(texts[i])
                        if np.max(np.abs(sv.amplitudes() - refs[i])) > 1e-10:
                            errors.append((tid, i))
                        sv.init_zero()
                        sv.apply_circuit(shared)
                        if np.max(np.abs(sv.amplitudes() - ref_shared)) > 1e-10:
                            errors.append((tid, "shared"))
        except Exception as e:  # noqa: BLE001
            errors.append((tid, repr(e)))

    th = [threading.Thread(target=work, args=(i,)) for i in range(4)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors, errors[:5]


@pytest.mark.gpu
def test_32q_mirror_with_top_tile_qubit(P):
    """32 qubits on one GPU (complex64, 32 GiB): a tile containing qubit 31 takes the widest
    32-bit tile-base computation (jit.cpp; no shift by 32); the circuit and its inverse return
    |0...0> (mirror)."""
    c = W.supremacy(7, 5, 20, 0, n=32)
    plan = P.Plan(W.to_text(c), "c64")
    assert any("b32_&=" in plan.source(i) for i in range(plan.info()["passes"]))
    m = W.concat(c, W.inverse(c))
    with P.StateVector(32, "c64") as sv:
        sv.apply_circuit(W.to_text(m))
        a = sv.amplitudes(0, 4)
        nrm = sv.norm()
    assert abs(a[0] - 1) < 1e-3 and np.max(np.abs(a[1:])) < 1e-4 and abs(nrm - 1) < 1e-3
