"""Pins for the CPU oracle (oracle/sv_oracle.c) against what the paper and mathematics fix.

Nothing here compares the oracle with itself: every expected value comes from an
independent formulation (brute-force matrices in tests/brute.py), a closed form, an
invariant, or a value printed in the paper/SPEC (tests/golden/paper_values.json).
"""

import json
import os

import numpy as np
import pytest

import oracle
import workloads as W
from tests import brute

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))


# ------------------------------------------------------------------ the test's own table
def test_brute_table_identities():
    """The brute-force gate table obeys the algebra that defines the gates (App. A, R3)."""
    T = brute.TABLE
    X, Y, Z = T["X"][1], T["Y"][1], T["Z"][1]
    assert np.allclose(T["SqrtX"][1] @ T["SqrtX"][1], X, atol=1e-15)
    assert np.allclose(T["SqrtY"][1] @ T["SqrtY"][1], Y, atol=1e-15)
    assert np.allclose(T["T"][1] @ T["T"][1], T["S"][1], atol=1e-15)
    assert np.allclose(T["S"][1] @ T["S"][1], Z, atol=1e-15)
    assert np.allclose(T["H"][1] @ Z @ T["H"][1], X, atol=1e-15)
    assert np.allclose(X @ Y, 1j * Z)
    for name, (_, U) in T.items():
        assert np.allclose(U.conj().T @ U, np.eye(U.shape[0]), atol=1e-12), name


# ------------------------------------------------------------------ brute force, n <= 8
@pytest.mark.parametrize("seed", range(12))
def test_oracle_matches_bruteforce_random(seed):
    """SURVEY 8(c) pin 1: full 2^n x 2^n embedded products vs the oracle, all gate kinds."""
    rng = np.random.default_rng(1000 + seed)
    n = int(rng.integers(3, 9))
    c = W.random_circuit(n, 40, seed, max_k=3, max_controls=2)
    psi0 = W.random_state(n, seed)
    ref = brute.simulate(c, psi0)
    got = oracle.simulate(W.to_text(c), psi0)
    assert np.max(np.abs(got - ref)) <= 1e-12


def test_oracle_k4_k5_blocks():
    rng = np.random.default_rng(7)
    for k in (4, 5):
        n = 7
        U = W.circuits.random_unitary(k, rng)
        tg = [int(x) for x in rng.choice(n, k, replace=False)]
        psi0 = W.random_state(n, k)
        ref = brute.embed(n, U, tg) @ psi0
        got = oracle.apply_gate(psi0.copy(), U, tg)
        assert np.max(np.abs(got - ref)) <= 1e-12


def test_oracle_controlled_unsorted_targets():
    """R22: control above target, unsorted target lists, k = n."""
    rng = np.random.default_rng(3)
    n = 5
    psi0 = W.random_state(n, 3)
    U = W.circuits.random_unitary(2, rng)
    got = oracle.apply_gate(psi0.copy(), U, [4, 1], [3, 0])
    ref = brute.embed(n, U, (4, 1), (3, 0)) @ psi0
    assert np.max(np.abs(got - ref)) <= 1e-13
    U5 = W.circuits.random_unitary(5, rng)
    got = oracle.apply_gate(psi0.copy(), U5, [2, 0, 4, 1, 3])
    ref = brute.embed(n, U5, (2, 0, 4, 1, 3)) @ psi0
    assert np.max(np.abs(got - ref)) <= 1e-12


# ------------------------------------------------------------------ closed forms
@pytest.mark.parametrize("n", [1, 2, 5, 12])
def test_hadamard_layer_is_uniform(n):
    """H on every qubit of |0> gives 2^(-n/2) everywhere (not bit-exact)."""
    txt = f"qubits: {n}\n" + "; ".join(f"H {q}" for q in range(n)) + "\n"
    psi = oracle.simulate(txt)
    assert np.max(np.abs(psi - 2.0 ** (-n / 2))) <= 1e-12
    assert np.max(np.abs(psi - oracle.uniform_state(n))) <= 1e-12


def test_uniform_golden():
    for row in GOLDEN["uniform_amplitude"]:
        psi = oracle.uniform_state(row["n"])
        assert psi[0].real == row["value"] and np.all(psi == psi[0]), row["cite"]
    assert oracle.norm(oracle.uniform_state(8)) == pytest.approx(1.0, abs=1e-12)


@pytest.mark.parametrize("k", [0, 3, 6])
def test_x_moves_unit_amplitude(k):
    """X on qubit k of |0> -> unit amplitude at index 2^k, exactly."""
    psi = oracle.simulate(f"qubits: 7\nX {k}\n")
    expect = np.zeros(128, complex)
    expect[1 << k] = 1
    assert np.array_equal(psi, expect)


def test_spec_kernel_examples():
    # S:175 CNOT(control 0, target 1) on |01> (index 1) -> index 3
    psi = oracle.simulate("qubits: 2\nX 0\nCNOT 0,1\n")
    assert psi[3] == 1 and np.count_nonzero(psi) == 1
    # S:120 H on q0 of |00>: amp[1] = 0.7071067811865476
    psi = oracle.simulate("qubits: 2\nH 0\n")
    assert abs(psi[1] - GOLDEN["h_on_q0_amp1"]["value"]) <= 1e-15
    # S:176 T on q2 of uniform(3): bit-2-set amplitudes times e^{i pi/4}
    u = oracle.uniform_state(3)
    psi = oracle.simulate("qubits: 3\nT 2\n", u)
    for i in range(8):
        f = np.exp(1j * np.pi / 4) if (i >> 2) & 1 else 1
        assert abs(psi[i] - u[i] * f) <= 1e-15
    # S:205 H.H = I
    psi = oracle.simulate("qubits: 1\nH 0\nH 0\n")
    assert abs(psi[0] - 1) <= 1e-15 and abs(psi[1]) <= 1e-15
    # S:184 identity Custom gate leaves the state unchanged exactly
    u = W.random_state(4, 1)
    psi = oracle.simulate("qubits: 4\nU 2,0 : " + ",".join(
        "1.0,0.0" if r == c else "0.0,0.0" for r in range(4) for c in range(4)) + "\n", u)
    assert np.array_equal(psi, u)
    # S:204 empty circuit
    assert np.array_equal(oracle.simulate("qubits: 3\n", u[:8] * 0 + 1), np.ones(8))


@pytest.mark.parametrize("n,k", [(5, 0), (5, 1), (5, 6), (5, 19), (5, 31), (9, 300), (12, 2741)])
def test_qft_closed_form(n, k):
    """QFT|k> = 2^(-n/2) sum_j e^{+2 pi i jk / 2^n} |j> (little-endian)."""
    c = W.concat(W.basis_prep(W.Circuit(n, []), k), W.qft(n))
    psi = oracle.simulate(W.to_text(c))
    j = np.arange(1 << n)
    expect = np.exp(2j * np.pi * j * k / (1 << n)) / np.sqrt(1 << n)
    assert np.max(np.abs(psi - expect)) <= 1e-12


def test_mirror_round_trip():
    """C then C^dagger returns psi_in."""
    c = W.supremacy(3, 3, 8, seed=5)
    psi0 = W.random_state(9, 5)
    psi = oracle.simulate(W.to_text(W.concat(c, W.inverse(c))), psi0)
    assert np.max(np.abs(psi - psi0)) <= 1e-12


def test_norm_preserved_supremacy():
    """|norm - 1| <= 1e-9 after a benchmark circuit."""
    psi = oracle.simulate(W.to_text(W.supremacy(4, 4, 12, seed=2)))
    assert abs(oracle.norm(psi) - 1) <= 1e-9


def test_supremacy_vs_bruteforce():
    c = W.supremacy(4, 2, 10, seed=4)
    assert np.max(np.abs(oracle.simulate(W.to_text(c)) - brute.simulate(c))) <= 1e-12


# ------------------------------------------------------------------ norm / readout
def test_norm_values():
    assert oracle.norm(oracle.zero_state(5)) == 1.0
    assert oracle.norm(np.zeros(16, complex)) == 0.0
    v = np.zeros(4, complex)
    v[:] = [3, 4j, 0, 0]
    assert oracle.norm(v) == 5.0


def test_probabilities_marginal():
    psi = W.random_state(6, 11)
    p = np.abs(psi) ** 2
    qs = [4, 1, 5]
    got = oracle.probabilities(psi, qs)
    # independent: reshape to a rank-6 tensor (axis a <-> qubit 5-a) and sum out the rest
    t = p.reshape([2] * 6)
    axes_keep = [5 - q for q in qs]
    other = tuple(a for a in range(6) if a not in axes_keep)
    m = t.sum(axis=other)  # remaining axes in increasing axis order
    kept_sorted = sorted(axes_keep)
    ref = np.zeros(8)
    for kidx in range(8):
        idx = [0] * 3
        for j, q in enumerate(qs):
            idx[kept_sorted.index(5 - q)] = (kidx >> j) & 1
        ref[kidx] = m[tuple(idx)]
    assert np.max(np.abs(got - ref)) <= 1e-15
    assert abs(oracle.probabilities(psi, list(range(6))) - p).max() <= 1e-16


def test_memory_estimate_golden():
    for row in GOLDEN["memory_estimate_bytes"]:
        assert oracle.memory_estimate(row["n"], row["bytes_per_amp"]) == row["value"], row["cite"]
    for n in range(1, 40):
        assert oracle.memory_estimate(n + 1) == 2 * oracle.memory_estimate(n)
    assert oracle.memory_estimate(60, 16) == 2 ** 64 - 1  # R20 saturation
    assert oracle.memory_estimate(30, 8) == 2 ** 33


# ------------------------------------------------------------------ multiplier (exact)
@pytest.mark.parametrize("nbits", [1, 2, 3])
def test_multiplier_exhaustive(nbits):
    """for all (a,b), |a,b,0,0> -> |a,b,ab,0> with amplitude exactly 1."""
    c = W.multiplier(nbits)
    n = c.n
    assert n == 4 * nbits + 1
    text = W.to_text(c)
    for a in range(1 << nbits):
        for b in range(1 << nbits):
            psi = oracle.zero_state(n) * 0
            psi[a | (b << nbits)] = 1
            out = oracle.simulate(text, psi)
            idx = a | (b << nbits) | ((a * b) << (2 * nbits))
            expect = np.zeros(1 << n, complex)
            expect[idx] = 1
            assert np.array_equal(out, expect), (a, b)


def test_multiplier_classical_map_n5_all_pairs():
    """Config 2 (21q, n=5): all 1024 basis inputs via the oracle's bit-level evaluator."""
    c = W.multiplier(5)
    ins = np.array([a | (b << 5) for a in range(32) for b in range(32)], dtype=np.uint64)
    outs = oracle.classical_map(W.to_text(c), ins)
    expect = np.array([a | (b << 5) | ((a * b) << 10) for a in range(32) for b in range(32)], np.uint64)
    assert np.array_equal(outs, expect)


def test_multiplier_rect_8x7_sampled():
    c = W.multiplier(8, 7)
    assert c.n == 31
    rng = np.random.default_rng(0)
    a = rng.integers(0, 256, 500)
    b = rng.integers(0, 128, 500)
    ins = (a | (b << 8)).astype(np.uint64)
    outs = oracle.classical_map(W.to_text(c), ins)
    assert np.array_equal(outs, (a | (b << 8) | ((a * b) << 15)).astype(np.uint64))


def test_classical_map_agrees_with_amplitudes():
    """Permutation circuits: psi_out[f(i)] == psi_in[i] exactly."""
    c = W.multiplier(2)
    text = W.to_text(c)
    psi0 = W.random_state(c.n, 9)
    out = oracle.simulate(text, psi0)
    f = oracle.classical_map(text, np.arange(1 << c.n, dtype=np.uint64))
    assert np.array_equal(out[f.astype(np.int64)], psi0)
    with pytest.raises(oracle.OracleError):
        oracle.classical_map("qubits: 2\nH 0\n", np.arange(4, dtype=np.uint64))


def _py_reversible(gates, x):
    """Brute-force classical evaluation, one bit at a time (independent of the oracle):
    ("x", controls, t) flips bit t when every control bit is 1; ("swap", controls, a, b)
    exchanges bits a and b when every control bit is 1."""
    for g in gates:
        if not all((x >> c) & 1 for c in g[1]):
            continue
        if g[0] == "x":
            x ^= 1 << g[2]
        else:
            a, b = g[2], g[3]
            if ((x >> a) ^ (x >> b)) & 1:
                x ^= (1 << a) | (1 << b)
    return x


def _reversible_text(n, gates):
    sw = "1,0,0,0,0,0,0,0,0,0,0,0,1,0,0,0,0,0,1,0,0,0,0,0,0,0,0,0,0,0,1,0"  # SWAP, interleaved re,im
    lines = [f"qubits: {n}"]
    for g in gates:
        if g[0] == "x":
            name = {0: "X", 1: "CNOT", 2: "Toffoli"}.get(len(g[1]))
            if name:
                lines.append(f"{name} " + ",".join(str(q) for q in (*g[1], g[2])))
            else:
                lines.append(f"CU {','.join(map(str, g[1]))}|{g[2]} : 0,0,1,0,1,0,0,0")
        elif not g[1]:
            lines.append(f"SWAP {g[2]},{g[3]}")
        else:
            lines.append(f"CU {','.join(map(str, g[1]))}|{g[2]},{g[3]} : {sw}")
    return "\n".join(lines) + "\n"


@pytest.mark.parametrize("seed", range(4))
def test_classical_map_range_brute_force(seed):
    """SURVEY 8(c) step 5's bit-sliced evaluator (or_classical_map_range) against a bit-by-bit
    Python evaluation over every input of random X / CNOT / Toffoli / multi-controlled X /
    SWAP / Fredkin circuits (n = 9), and against the per-index or_classical_map."""
    rng = np.random.default_rng(100 + seed)
    n = 9
    gates = []
    for _ in range(60):
        kind = rng.integers(0, 2)
        nctl = int(rng.integers(0, 4))
        qs = [int(q) for q in rng.permutation(n)[: nctl + 2]]
        gates.append(("x", qs[:nctl], qs[nctl]) if kind == 0 else ("swap", qs[:nctl], qs[nctl], qs[nctl + 1]))
    text = _reversible_text(n, gates)
    got = oracle.classical_map_range(text, 0, 1 << n)
    expect = np.array([_py_reversible(gates, x) for x in range(1 << n)], dtype=np.uint64)
    assert np.array_equal(got, expect)
    assert np.array_equal(got, oracle.classical_map(text, np.arange(1 << n, dtype=np.uint64)))
    # a sub-range at an offset gives the same values
    assert np.array_equal(oracle.classical_map_range(text, 128, 192), expect[128:320])


def test_classical_map_range_multiplier_products():
    """The 31 q 8x7 multiplier over a 2^16 range of inputs with an empty product register:
    (a, b, 0, 0) -> (a, b, a*b, 0) (closed form), and an arbitrary range equals the per-index map."""
    c = W.multiplier(8, 7)
    text = W.to_text(c)
    got = oracle.classical_map_range(text, 0, 1 << 15)
    x = np.arange(1 << 15, dtype=np.uint64)
    a, b = x & 255, x >> 8
    assert np.array_equal(got, a | (b << 8) | ((a * b) << 15))
    first = (123457 << 6) * 977 & ((1 << 31) - 1) & ~63
    got = oracle.classical_map_range(text, first, 4096)
    assert np.array_equal(got, oracle.classical_map(text, np.arange(first, first + 4096, dtype=np.uint64)))
    with pytest.raises(oracle.OracleError):
        oracle.classical_map_range("qubits: 7\nH 0\n", 0, 128)
    with pytest.raises(oracle.OracleError):
        oracle.classical_map_range(text, 3, 64)


# ------------------------------------------------------------------ determinism, errors
def test_thread_count_bit_identical():
    """bit-identical for any worker count."""
    text = W.to_text(W.supremacy(4, 4, 8, seed=1))
    a = oracle.simulate(text, nthreads=1)
    b = oracle.simulate(text, nthreads=4)
    assert np.array_equal(a, b)


@pytest.mark.parametrize("text,line", [
    ("qubits: 3\nH 0\nFOO 1\n", 3),
    ("qubits: 3\nH 0; CNOT 1\n", 2),
    ("qubits: 3\n\nH 5\n", 3),
    ("qubits: 3\nCZ 1,1\n", 2),
    ("H 0\n", 1),
    ("qubits: 2\nU 0 : 1,0,0,0\n", 2),
])
def test_parse_errors_name_line(text, line):
    with pytest.raises(oracle.OracleError, match=f"line {line}"):
        oracle.circuit_info(text)
