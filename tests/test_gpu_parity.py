"""GPU path vs the CPU oracle, element by element, through the C-ABI (libsv.so).

Tolerances (written here): north_star max|d amplitude| <= 1e-10 (c128),
<= 1e-4 (c64), plus ||d||_2 <= 8 G u (reading R9); bit-exact (==) for basis-input
permutation circuits (reading R10).  c64 runs feed both sides the c64-rounded input.
"""

import numpy as np
import pytest

import oracle
import workloads as W
from tests.parity import assert_close

pytestmark = pytest.mark.gpu

MODES = {"fused": {}, "per_gate": {"fuse": False}, "dense": {"force_kernel": 2}}


@pytest.fixture(scope="module")
def P():
    import paper_2106_13995_b200 as P
    return P


def run_gpu(P, text, n, dtype, psi0=None, init=None, **opts):
    with P.StateVector(n, dtype) as sv:
        if psi0 is not None:
            sv.set_amplitudes(psi0)
        elif init == "uniform":
            sv.init_uniform()
        st = sv.apply_circuit(text, **opts)
        return sv.amplitudes(), st


def input_for(n, seed, dtype):
    psi = W.random_state(n, seed)
    return W.round_to_c64(psi) if dtype == "c64" else psi


# ------------------------------------------------------------------ random circuits, all kinds
@pytest.mark.parametrize("mode", list(MODES))
@pytest.mark.parametrize("dtype", ["c128", "c64"])
@pytest.mark.parametrize("seed", range(8))
def test_random_circuits(P, seed, dtype, mode):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(2, 15))
    c = W.random_circuit(n, 80, seed, max_k=min(5, n), max_controls=2)
    text = W.to_text(c)
    psi0 = input_for(n, seed, dtype)
    got, st = run_gpu(P, text, n, dtype, psi0, **MODES[mode])
    ref = oracle.simulate(text, psi0)
    assert st["gates"] == W.gate_count(c)
    assert_close(got, ref, dtype, W.gate_count(c))


@pytest.mark.parametrize("dtype", ["c128", "c64"])
@pytest.mark.parametrize("n", [1, 2, 3, 5, 6, 9, 13, 14, 17])
def test_every_named_gate_every_position(P, n, dtype):
    """Each named kind on every qubit (register bits, lane bits, tile bits, tile base bits)."""
    gates = []
    rng = np.random.default_rng(n)
    for name, ar in W.circuits.ARITY.items():
        if ar > n:
            continue
        for q in range(n):
            qs = [q] + [int(x) for x in rng.choice([p for p in range(n) if p != q], ar - 1, replace=False)]
            gates.append(W.GateSpec(name, tuple(qs[1:] + qs[:1]) if ar > 1 else (q,)))
    c = W.Circuit(n, [[g] for g in gates])
    text = W.to_text(c)
    psi0 = input_for(n, 100 + n, dtype)
    ref = oracle.simulate(text, psi0)
    for mode in MODES.values():
        got, _ = run_gpu(P, text, n, dtype, psi0, **mode)
        assert_close(got, ref, dtype, len(gates))


@pytest.mark.parametrize("dtype", ["c128", "c64"])
def test_wide_blocks_and_controls(P, dtype):
    """U3/U4/U5 blocks with unsorted targets and controls inside and outside the tile."""
    n = 16
    rng = np.random.default_rng(5)
    gates = []
    for k in (2, 3, 4, 5):
        for _ in range(4):
            qs = [int(x) for x in rng.choice(n, k + 2, replace=False)]
            U = W.circuits.random_unitary(k, rng)
            gates.append(W.GateSpec("CU", tuple(qs[2:]), tuple(qs[:2]), tuple(complex(x) for x in U.reshape(-1))))
            gates.append(W.GateSpec("U", tuple(qs[:k]), (), tuple(complex(x) for x in U.conj().T.reshape(-1))))
    c = W.Circuit(n, [[g] for g in gates])
    text = W.to_text(c)
    psi0 = input_for(n, 5, dtype)
    ref = oracle.simulate(text, psi0)
    for mode in MODES.values():
        got, _ = run_gpu(P, text, n, dtype, psi0, **mode)
        assert_close(got, ref, dtype, len(gates))


# ------------------------------------------------------------------ config 1: 12q supremacy d10 c128
@pytest.mark.parametrize("seed", range(5))
def test_config1_supremacy_12q(P, seed):
    c = W.supremacy(4, 3, 10, seed)
    text = W.to_text(c)
    ref = oracle.simulate(text)
    for mode in MODES.values():
        got, _ = run_gpu(P, text, 12, "c128", **mode)
        assert_close(got, ref, "c128", W.gate_count(c))


@pytest.mark.parametrize("dtype", ["c128", "c64"])
def test_supremacy_20q_vs_oracle(P, dtype):
    c = W.supremacy(5, 4, 14, seed=3)
    text = W.to_text(c)
    ref = oracle.simulate(text)
    got, st = run_gpu(P, text, 20, dtype)
    assert_close(got, ref, dtype, W.gate_count(c))
    assert st["passes"] < W.gate_count(c) / 4  # fusion really fuses


def test_qft_closed_form_gpu(P):
    n, k = 15, 12345
    c = W.concat(W.basis_prep(W.Circuit(n, []), k), W.qft(n))
    got, _ = run_gpu(P, W.to_text(c), n, "c128")
    j = np.arange(1 << n)
    expect = np.exp(2j * np.pi * j * k / (1 << n)) / np.sqrt(1 << n)
    assert np.max(np.abs(got - expect)) <= 1e-12


def phase_heavy_circuit(n, ngates, seed):
    """Controlled phases (QFT-style), single-qubit diagonals with a global part, controlled
    1-qubit phases, interleaved with H, SqrtX, X, SWAP, CNOT and dense 2-qubit U: every kind
    of term of the generator's pending phase polynomial, with register, thread and tile-base
    partners."""
    rng = np.random.default_rng(seed)
    gates = []
    for _ in range(ngates):
        r = rng.random()
        th = float(rng.uniform(0, 2 * np.pi))
        if r < 0.35:
            a, b = (int(x) for x in rng.choice(n, 2, replace=False))
            m = np.diag([1, 1, 1, np.exp(1j * th)])
            gates.append(W.GateSpec("U", (a, b), (), tuple(complex(x) for x in m.reshape(-1))))
        elif r < 0.5:
            a, b = (int(x) for x in rng.choice(n, 2, replace=False))
            m = np.diag([1, np.exp(1j * th)])
            gates.append(W.GateSpec("CU", (a,), (b,), tuple(complex(x) for x in m.reshape(-1))))
        elif r < 0.6:
            a = int(rng.integers(n))
            m = np.diag([np.exp(1j * th), np.exp(1j * float(rng.uniform(0, 2 * np.pi)))])
            gates.append(W.GateSpec("U", (a,), (), tuple(complex(x) for x in m.reshape(-1))))
        elif r < 0.9:
            name = ["H", "SqrtX", "X", "H", "T"][int(rng.integers(5))]
            gates.append(W.GateSpec(name, (int(rng.integers(n)),)))
        elif r < 0.95:
            a, b = (int(x) for x in rng.choice(n, 2, replace=False))
            gates.append(W.GateSpec(["SWAP", "CNOT"][int(rng.integers(2))], (a, b)))
        else:
            a, b = (int(x) for x in rng.choice(n, 2, replace=False))
            m = W.random_unitary(2, rng)
            gates.append(W.GateSpec("U", (a, b), (), tuple(complex(x) for x in m.reshape(-1))))
    return W.Circuit(n, [[g] for g in gates], "custom", {"seed": seed})


@pytest.mark.parametrize("dtype", ["c128", "c64"])
@pytest.mark.parametrize("n,seed", [(6, 0), (14, 1), (17, 2), (20, 3)])
def test_phase_polynomial_circuits(P, dtype, n, seed):
    c = phase_heavy_circuit(n, 300, seed)
    text = W.to_text(c)
    psi0 = input_for(n, seed + 10, dtype)
    ref = oracle.simulate(text, psi0)
    for mode in ({}, {"fuse": False}):
        got, _ = run_gpu(P, text, n, dtype, psi0=psi0, **mode)
        assert_close(got, ref, dtype, W.gate_count(c))


@pytest.mark.parametrize("dtype", ["c128", "c64"])
@pytest.mark.parametrize("n,seed", [(4, 0), (15, 1), (21, 2)])
def test_merged_single_qubit_runs(P, dtype, n, seed):
    # runs of unit-class 1-qubit gates merged by the planner (merge_single_qubit), incl. custom
    # U with a global phase; fused and per-gate (unmerged lowering of single gates) both
    from tests.test_generator_cpu import clifford_run_circuit
    c = clifford_run_circuit(n, 400, seed)
    text = W.to_text(c)
    psi0 = input_for(n, seed + 30, dtype)
    ref = oracle.simulate(text, psi0)
    for mode in ({}, {"fuse": False}):
        got, _ = run_gpu(P, text, n, dtype, psi0=psi0, **mode)
        assert_close(got, ref, dtype, W.gate_count(c))


@pytest.mark.parametrize("dtype", ["c128", "c64"])
def test_deferred_uniform_init(P, dtype):
    # sv_init_uniform on one GPU is deferred: the plan's first tile pass synthesises 2^(-n/2)
    # instead of reading (tile pass and permutation plans), any other call writes it first
    for c in (W.supremacy(4, 4, 8, seed=5, n=16), W.multiplier(4)):
        text = W.to_text(c)
        nn = c.n
        uu = np.full(1 << nn, 2.0 ** (-nn / 2), complex)
        ref = oracle.simulate(text, uu)
        plan = P.Plan(text, dtype)
        with P.StateVector(nn, dtype) as sv:
            for _ in range(2):
                sv.init_uniform()
                sv.apply_plan(plan)
                assert_close(sv.amplitudes(), ref, dtype, W.gate_count(c))
            sv.init_uniform()
            got = sv.amplitudes()  # materialised by the readout
            assert np.max(np.abs(got - uu)) <= (1e-7 if dtype == "c64" else 1e-15)
            sv.init_uniform()
            sv.apply_gate(np.array([[1, 0], [0, -1]]), [0])  # materialised before a single gate
            z = uu.copy()
            z[1::2] *= -1
            assert np.max(np.abs(sv.amplitudes() - z)) <= (1e-7 if dtype == "c64" else 1e-15)


def test_qft_20q_vs_oracle(P):
    c = W.qft(20)
    text = W.to_text(c)
    psi0 = input_for(20, 4, "c128")
    ref = oracle.simulate(text, psi0)
    for dtype in ("c128", "c64"):
        got, st = run_gpu(P, text, 20, dtype, psi0=input_for(20, 4, dtype))
        assert_close(got, oracle.simulate(text, input_for(20, 4, dtype)) if dtype == "c64" else ref, dtype,
                     W.gate_count(c))


# ------------------------------------------------------------------ config 2: multiplier, basis inputs
def test_config2_multiplier_21q_bit_exact(P):
    c = W.multiplier(5)
    text = W.to_text(c)
    n = c.n
    plan = P.Plan(text, "c128")
    # two full-state comparisons against the oracle, bit for bit
    for a, b in [(19, 27), (31, 31)]:
        x = a | (b << 5)
        psi0 = np.zeros(1 << n, complex)
        psi0[x] = 1
        ref = oracle.simulate(text, psi0)
        with P.StateVector(n, "c128") as sv:
            sv.init_basis(x)
            sv.apply_plan(plan)
            got = sv.amplitudes()
        assert np.array_equal(got, ref)
    # all 1024 pairs: amplitude exactly 1 at the oracle's classical image, norm exactly 1
    ins = np.array([a | (b << 5) for a in range(32) for b in range(32)], dtype=np.uint64)
    outs = oracle.classical_map(text, ins)
    with P.StateVector(n, "c128") as sv:
        for x, y in zip(ins.tolist(), outs.tolist()):
            sv.init_basis(x)
            sv.apply_plan(plan)
            amp = sv.amplitudes(int(y), 1)[0]
            assert amp == 1 + 0j and sv.norm() == 1.0, (x, y, amp)
            a, b = x & 31, x >> 5
            assert y == x | ((a * b) << 10)


@pytest.mark.parametrize("dtype", ["c64", "c128"])
def test_permutation_pass_random_state_exact(P, dtype):
    """a reversible circuit runs as one gather pass; on any input the result
    is psi_out[f(i)] == psi_in[i] exactly (f from the oracle's bit-level evaluator)."""
    # a multiplier on qubits 3..15 (the low qubits stay put, so the gathers coalesce and the
    # planner picks the gather pass), basis preparation, and a SWAP
    m = W.multiplier(3)
    shifted = [[W.GateSpec(g.name, tuple(q + 3 for q in g.qubits)) for g in mom] for mom in m.moments]
    c = W.concat(W.basis_prep(W.Circuit(16, []), 0b1010011 << 3),
                 W.Circuit(16, shifted + [[W.GateSpec("SWAP", (15, 4))]]))
    text = W.to_text(c)
    plan = P.Plan(text, dtype)
    assert plan.info()["passes"] == 1 and "permutation pass" in plan.source(0)
    psi0 = input_for(16, 77, dtype)
    f = oracle.classical_map(text, np.arange(1 << 16, dtype=np.uint64)).astype(np.int64)
    with P.StateVector(16, dtype) as sv:
        sv.set_amplitudes(psi0)
        sv.apply_plan(plan)
        got = sv.amplitudes()
    assert np.array_equal(got[f], psi0.astype(got.dtype))
    assert np.array_equal(got.astype(complex), oracle.simulate(text, psi0))


def test_permutation_pass_borrowed_buffer(P):
    """A borrowed (torch) buffer gets the result copied back in place."""
    import torch
    c = W.multiplier(3)
    text = W.to_text(c)
    psi0 = W.random_state(13, 5)
    t = torch.tensor(psi0, dtype=torch.complex128, device="cuda")
    with P.StateVector.wrap(t, 13) as sv:
        sv.apply_circuit(text)
        sv.sync()
        got = t.cpu().numpy()
    assert np.array_equal(got, oracle.simulate(text, psi0))


def test_multiplier_superposition_support(P):
    """H on A and B: support exactly {|a,b,ab,0>}, each 2^-n (not bit-exact: H rounds)."""
    nb = 3
    c = W.multiplier(nb)
    h = W.Circuit(c.n, [[W.GateSpec("H", (q,)) for q in range(2 * nb)]])
    got, _ = run_gpu(P, W.to_text(W.concat(h, c)), c.n, "c128")
    expect = np.zeros(1 << c.n)
    for a in range(1 << nb):
        for b in range(1 << nb):
            expect[a | (b << nb) | ((a * b) << (2 * nb))] = 2.0 ** -nb
    assert np.max(np.abs(got - expect)) <= 1e-12


# ------------------------------------------------------------------ readout / init
@pytest.mark.parametrize("dtype", ["c128", "c64"])
def test_readout_probabilities_norm(P, dtype):
    n = 14
    c = W.supremacy(4, 3, 6, seed=1)
    c = W.Circuit(n, c.moments + [[W.GateSpec("H", (12,)), W.GateSpec("SqrtX", (13,))]])
    text = W.to_text(c)
    psi0 = input_for(n, 7, dtype)
    ref = oracle.simulate(text, psi0)
    with P.StateVector(n, dtype) as sv:
        sv.set_amplitudes(psi0)
        sv.apply_circuit(text)
        tol = 1e-12 if dtype == "c128" else 1e-5
        for qs in ([], [0], [13], [3, 0, 11], list(range(n)), [5, 6, 7, 8, 9, 10, 1]):
            got = sv.probabilities(qs)
            assert np.max(np.abs(got - oracle.probabilities(ref, qs))) <= tol, qs
        assert abs(sv.norm() - oracle.norm(ref)) <= tol


@pytest.mark.parametrize("dtype", ["c128", "c64"])
def test_wide_marginals_relabelled_layout(P, dtype):
    """Wide subsets (>= 12 qubits: the lane kernel) on a state left in a relabelled physical
    layout by the plan: orders, subsets without the low qubits, all qubits."""
    n = 20
    c = W.supremacy(5, 4, 12, seed=3)
    text = W.to_text(c)
    ref = oracle.simulate(text)
    rng = np.random.default_rng(5)
    subsets = [list(range(n)), list(range(4, 20)), list(range(19, 5, -1)),
               [int(x) for x in rng.permutation(n)[:14]], [0, 2, 4, 6, 8, 10, 12, 14, 16, 18, 1, 3]]
    tol = 1e-12 if dtype == "c128" else 1e-6
    with P.StateVector(n, dtype) as sv:
        sv.apply_circuit(text)
        assert sv.qubit_map() != list(range(n))  # the plan left a relabelled layout
        for qs in subsets:
            got = sv.probabilities(qs)
            assert np.max(np.abs(got - oracle.probabilities(ref, qs))) <= tol, qs
            assert np.array_equal(got, sv.probabilities(qs))  # deterministic


@pytest.mark.parametrize("dtype", ["c128", "c64"])
def test_fused_basis_init(P, dtype):
    """sv_init_basis is deferred and synthesised by the plan's first pass: same result, bit
    for bit, as the same plan run on the basis state written explicitly; readouts and
    single gates after an init see the written state."""
    n = 20
    for c in (W.supremacy(5, 4, 10, seed=4), W.multiplier(5)):
        text = W.to_text(c)
        plan = P.Plan(text, dtype)
        for k in (0, 1 << (c.n - 1), 0x5A5A5 & ((1 << c.n) - 1)):
            e = np.zeros(1 << c.n, np.complex128)
            e[k] = 1
            with P.StateVector(c.n, dtype) as a, P.StateVector(c.n, dtype) as b:
                a.init_basis(k)
                a.apply_plan(plan)
                b.set_amplitudes(e)
                b.apply_plan(plan)
                assert np.array_equal(a.amplitudes(), b.amplitudes()), (c.family, k)
    with P.StateVector(n, dtype) as sv:
        sv.init_basis(77)
        assert sv.amplitudes(77, 1)[0] == 1 and sv.norm() == 1
        sv.init_basis(5)
        p = sv.probabilities([0, 2])
        assert p[3] == 1
        sv.init_basis(6)
        sv.apply_gate(np.array([[0, 1], [1, 0]], complex), [0])
        assert sv.amplitudes(7, 1)[0] == 1


@pytest.mark.parametrize("dtype", ["c128", "c64"])
def test_init_states(P, dtype):
    for n in (1, 7, 20):
        with P.StateVector(n, dtype) as sv:
            a = sv.amplitudes()
            assert a[0] == 1 and np.count_nonzero(a) == 1
            sv.init_uniform()
            u = oracle.uniform_state(n)
            if dtype == "c64":
                u = W.round_to_c64(u)
            assert np.array_equal(sv.amplitudes().astype(complex), u)
            k = (1 << n) - 1 - (n // 3)
            sv.init_basis(k)
            a = sv.amplitudes()
            assert a[k] == 1 and np.count_nonzero(a) == 1


def test_apply_gate_api(P):
    n = 9
    rng = np.random.default_rng(2)
    psi0 = W.random_state(n, 2)
    U = W.circuits.random_unitary(2, rng)
    with P.StateVector(n, "c128") as sv:
        sv.set_amplitudes(psi0)
        sv.apply_gate(U, [7, 2], [4])
        got = sv.amplitudes()
    ref = oracle.apply_gate(psi0.copy(), U, [7, 2], [4])
    assert np.max(np.abs(got - ref)) <= 1e-13
    with P.StateVector(n, "c128") as sv:
        with pytest.raises(P.SvError, match="SV_ERR_RANGE"):
            sv.apply_gate(np.eye(2), [9])
        with pytest.raises(P.SvError, match="SV_ERR_RANGE"):
            sv.apply_gate(np.eye(4), [1, 1])
        with pytest.raises(P.SvError, match="SV_ERR_ARG"):
            sv.apply_gate(np.eye(64), [0, 1, 2, 3, 4, 5])


def test_empty_circuit_and_identity(P):
    psi0 = W.random_state(6, 4)
    got, st = run_gpu(P, "qubits: 6\n", 6, "c128", psi0)
    assert np.array_equal(got, psi0) and st["passes"] == 0
    eye = ",".join("1.0,0.0" if r == c else "0.0,0.0" for r in range(4) for c in range(4))
    got, _ = run_gpu(P, f"qubits: 6\nU 5,2 : {eye}\n", 6, "c128", psi0)
    assert np.array_equal(got, psi0)  # identity Custom gate, exact


def test_determinism_bitwise(P):
    c = W.supremacy(5, 4, 10, seed=8)
    text = W.to_text(c)
    a, _ = run_gpu(P, text, 20, "c64")
    b, _ = run_gpu(P, text, 20, "c64")
    assert np.array_equal(a, b)
    with P.StateVector(20, "c64") as sv:
        sv.apply_circuit(text)
        n1 = sv.norm()
        assert all(sv.norm() == n1 for _ in range(3))


def test_cuda_graph_replay(P):
    c = W.supremacy(4, 4, 8, seed=2)
    text = W.to_text(c)
    ref = oracle.simulate(text)
    plan = P.Plan(text, "c128", use_graph=True)
    with P.StateVector(16, "c128") as sv:
        for _ in range(3):
            sv.init_zero()
            sv.apply_plan(plan)
            assert_close(sv.amplitudes(), ref, "c128", W.gate_count(c))
