"""The generated sm_100a pass kernels, executed on the host (tools/emulate.py: the CUDA source
translated to C++, one std::thread per CUDA thread, a std::barrier per __syncthreads), against
the oracle.  Covers the code generator without a GPU: relabelling stores, per-transition
swizzles, deferred factors, run-time signs, the phase polynomial, both dtypes.  The GPU tests
(tests/test_gpu_parity.py) run the same kernels on the B200."""

import numpy as np
import pytest

import oracle
import workloads as W
from tests.parity import assert_close
from tools.emulate import run_plan_on_host, to_logical

pytestmark = pytest.mark.cpu_emulation


@pytest.fixture(scope="module")
def P():
    import paper_2106_13995_b200 as P
    return P


def phase_heavy_circuit(n, ngates, seed):
    from tests.test_gpu_parity import phase_heavy_circuit as f
    return f(n, ngates, seed)


def _emulated(P, text, n, dtype, psi):
    plan = P.Plan(text, dtype)
    x = psi.astype(np.complex64 if dtype == "c64" else np.complex128)
    return run_plan_on_host(plan, x), plan


@pytest.mark.parametrize("dtype", ["c128", "c64"])
def test_supremacy_14q(P, dtype):
    c = W.supremacy(4, 4, 12, seed=2, n=14)
    text = W.to_text(c)
    psi = W.random_state(14, 3)
    psi = W.round_to_c64(psi) if dtype == "c64" else psi
    got, plan = _emulated(P, text, 14, dtype, psi)
    assert plan.info()["passes"] >= 2
    assert_close(got, oracle.simulate(text, psi), dtype, W.gate_count(c))


@pytest.mark.parametrize("dtype", ["c128", "c64"])
@pytest.mark.parametrize("n,seed", [(6, 0), (14, 1)])
def test_phase_polynomial(P, dtype, n, seed):
    c = phase_heavy_circuit(n, 200, seed)
    text = W.to_text(c)
    psi = W.random_state(n, seed + 10)
    psi = W.round_to_c64(psi) if dtype == "c64" else psi
    got, _ = _emulated(P, text, n, dtype, psi)
    assert_close(got, oracle.simulate(text, psi), dtype, W.gate_count(c))


def test_qft_closed_form(P):
    n, k = 13, 4321
    c = W.concat(W.basis_prep(W.Circuit(n, []), k), W.qft(n))
    psi = np.zeros(1 << n, complex)
    psi[0] = 1
    got, _ = _emulated(P, W.to_text(c), n, "c128", psi)
    j = np.arange(1 << n)
    assert np.max(np.abs(got - np.exp(2j * np.pi * j * k / (1 << n)) / np.sqrt(1 << n))) <= 1e-12


@pytest.mark.parametrize("dtype", ["c128", "c64"])
def test_diagonal_heavy(P, dtype):
    """General 1- and 2-qubit diagonals (phase-polynomial terms incl. their global part)."""
    n = 13
    c = W.random_circuit(n, 80, 7, kinds=["Udiag", "H", "SqrtX", "CNOT", "T", "CZ"], max_k=2, max_controls=1)
    text = W.to_text(c)
    psi = W.random_state(n, 7)
    psi = W.round_to_c64(psi) if dtype == "c64" else psi
    got, _ = _emulated(P, text, n, dtype, psi)
    assert_close(got, oracle.simulate(text, psi), dtype, W.gate_count(c))


@pytest.mark.parametrize("seed", range(3))
def test_random_circuits(P, seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(9, 14))
    c = W.random_circuit(n, 60, seed, max_k=4, max_controls=2)
    text = W.to_text(c)
    psi = W.random_state(n, seed)
    plan = P.Plan(text, "c128")
    srcs = [plan.source(i) for i in range(plan.info()["passes"])]
    if not all(srcs):
        pytest.skip("plan has a non-tile pass")
    got = run_plan_on_host(plan, psi)
    assert_close(got, oracle.simulate(text, psi), "c128", W.gate_count(c))


def test_to_logical_roundtrip():
    n = 5
    qmap = [3, 0, 4, 1, 2]
    x = np.arange(1 << n) + 0j
    # physical index of logical i
    phys = np.zeros(1 << n, np.int64)
    for i in range(1 << n):
        phys[i] = sum(((i >> q) & 1) << qmap[q] for q in range(n))
    y = np.zeros_like(x)
    y[phys] = x
    assert np.array_equal(to_logical(y, qmap, n), x)


def clifford_run_circuit(n, ngates, seed):
    """Long same-qubit runs of unit-class 1-qubit gates (Paulis, H, S, SqrtX/SqrtY and inverses,
    and unit-class custom U with a global phase), mixed with T and CZ -- the runs the planner
    merges into one butterfly or one permutation/phase (planner.cpp merge_single_qubit)."""
    rng = np.random.default_rng(seed)
    one = ["X", "Y", "Z", "H", "S", "Sdg", "SqrtX", "SqrtY", "SqrtXdg", "SqrtYdg"]
    gates = []
    for _ in range(ngates):
        u = rng.random()
        if u < 0.08:
            a, b = (int(x) for x in rng.choice(n, 2, replace=False))
            gates.append(W.GateSpec("CZ", (a, b)))
        elif u < 0.14:
            gates.append(W.GateSpec("T", (int(rng.integers(n)),)))
        elif u < 0.24:
            ph = np.exp(1j * rng.uniform(0, 2 * np.pi))
            m = ph * np.array([[1, 1j], [1j, 1]]) / np.sqrt(2) if rng.random() < 0.5 else ph * np.array([[0, 1j], [1, 0]])
            gates.append(W.GateSpec("U", (int(rng.integers(n)),), (), tuple(complex(x) for x in m.reshape(-1))))
        else:
            # bias towards a few qubits so that long runs form
            q = int(rng.integers(min(n, 3))) if rng.random() < 0.6 else int(rng.integers(n))
            gates.append(W.GateSpec(one[rng.integers(len(one))], (q,)))
    return W.Circuit(n, [[g] for g in gates], "custom", {"seed": seed})


@pytest.mark.parametrize("dtype", ["c128", "c64"])
@pytest.mark.parametrize("n,seed", [(5, 0), (13, 1)])
def test_merged_single_qubit_runs(P, dtype, n, seed):
    c = clifford_run_circuit(n, 300, seed)
    text = W.to_text(c)
    psi = W.random_state(n, seed + 20)
    psi = W.round_to_c64(psi) if dtype == "c64" else psi
    got, _ = _emulated(P, text, n, dtype, psi)
    assert_close(got, oracle.simulate(text, psi), dtype, W.gate_count(c))


@pytest.mark.parametrize("dtype", ["c128", "c64"])
@pytest.mark.parametrize("k", [0, 5, 12345])
def test_basis_input_variant(P, dtype, k, monkeypatch):
    """The first pass's fused-init variant (synthesises |k> in registers) gives bit for bit
    what the generic pass gives on a stored |k>; the whole plan matches the oracle."""
    from tools.emulate import run_pass_on_host
    n = 14
    c = W.supremacy(4, 4, 12, seed=5, n=n)
    text = W.to_text(c)
    plan = P.Plan(text, dtype)
    cdt = np.complex64 if dtype == "c64" else np.complex128
    generic = plan.source(0)
    monkeypatch.setenv("SV_SOURCE_VARIANT", "basis")
    fused = plan.source(0)
    monkeypatch.delenv("SV_SOURCE_VARIANT")
    assert fused != generic and "kb" in fused
    a = np.zeros(1 << n, dtype=cdt)
    a[k] = 1
    run_pass_on_host(generic, a, n)
    b = np.full(1 << n, np.nan, dtype=cdt)  # the fused variant reads nothing
    run_pass_on_host(fused, b, n, basis=k)
    assert np.array_equal(a, b)
    # the rest of the plan after the fused first pass matches the oracle
    for i in range(1, plan.info()["passes"]):
        run_pass_on_host(plan.source(i), b, n)
    got = to_logical(b, plan.qubit_map(), n)
    psi = np.zeros(1 << n, dtype=np.complex128)
    psi[k] = 1
    assert_close(got, oracle.simulate(text, psi), dtype, W.gate_count(c))


@pytest.mark.parametrize("dtype", ["c64", "c128"])
@pytest.mark.parametrize("seed", range(4))
def test_supremacy_layouts_many_seeds(P, dtype, seed):
    """Wider coverage of the shared-memory layout search (additive offsets, XOR bases, 16-byte
    paired accesses, the barrier between a stage's reads and writes): supremacy circuits on
    grids whose plans take 4-low-position tiles (14 q and up, complex64) and several seeds,
    every pass executed on the host against the oracle."""
    rows, cols = [(4, 4), (5, 3), (7, 2), (4, 4)][seed]
    c = W.supremacy(rows, cols, 14, seed=10 + seed)
    text = W.to_text(c)
    psi = W.random_state(c.n, 20 + seed)
    psi = W.round_to_c64(psi) if dtype == "c64" else psi
    got, plan = _emulated(P, text, c.n, dtype, psi)
    assert plan.info()["passes"] >= 2
    assert_close(got, oracle.simulate(text, psi), dtype, W.gate_count(c))
