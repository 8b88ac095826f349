"""Generator pins: structure, widths, determinism, and the
multiplier's arithmetic checked by a classical bit simulator written here (independent of
both the oracle and the CUDA path)."""

import json
import os

import numpy as np
import pytest

import workloads as W

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))


def classical(gates, x):
    """Evaluate X/CNOT/Toffoli/SWAP on an integer bit string."""
    for g in gates:
        q = g.qubits
        if g.name == "X":
            x ^= 1 << q[0]
        elif g.name == "CNOT":
            if (x >> q[0]) & 1:
                x ^= 1 << q[1]
        elif g.name == "Toffoli":
            if (x >> q[0]) & 1 and (x >> q[1]) & 1:
                x ^= 1 << q[2]
        elif g.name == "SWAP":
            a, b = (x >> q[0]) & 1, (x >> q[1]) & 1
            if a != b:
                x ^= (1 << q[0]) | (1 << q[1])
        else:
            raise ValueError(g.name)
    return x


@pytest.mark.parametrize("na,nb", [(1, 1), (2, 2), (3, 3), (4, 4), (5, 5), (3, 2)])
def test_multiplier_arithmetic_exhaustive(na, nb):
    c = W.multiplier(na, nb)
    gates = c.gates
    for a in range(1 << na):
        for b in range(1 << nb):
            y = classical(gates, a | (b << na))
            assert y == a | (b << na) | ((a * b) << (na + nb)), (a, b)


@pytest.mark.parametrize("na,nb", [(7, 7), (8, 7), (8, 8)])
def test_multiplier_arithmetic_sampled(na, nb):
    c = W.multiplier(na, nb)
    rng = np.random.default_rng(na * 10 + nb)
    for _ in range(200):
        a, b = int(rng.integers(1 << na)), int(rng.integers(1 << nb))
        assert classical(c.gates, a | (b << na)) == a | (b << na) | ((a * b) << (na + nb))


def test_multiplier_counts_and_widths():
    for row in GOLDEN["multiplier_width"]:
        assert W.multiplier(row["operand_bits"]).n == row["width"], row["cite"]
    for n in range(1, 9):
        c = W.multiplier(n)
        assert W.gate_count(c) == n * (8 * n + 1)
        assert sum(g.name == "Toffoli" for g in c.gates) == n * (4 * n + 1)
        assert c.depth <= 9 * n * n  # S:304 depth O(n^2), c fitted at n=1..3
    assert W.gate_count(W.multiplier(8, 7)) == 455


def test_supremacy_structure():
    for row in GOLDEN["supremacy_width"]:
        assert W.supremacy(row["rows"], row["cols"], 2).n == row["width"], row["cite"]
    c = W.supremacy(6, 5, 20, seed=0)
    assert W.gate_count(c) == 507
    assert all(g.name == "H" for g in c.moments[0]) and len(c.moments[0]) == 30
    prev = {}
    for m in c.moments[1:]:
        for g in m:
            if g.name == "CZ":
                a, b = g.qubits
                ra, ca, rb, cb = a // 5, a % 5, b // 5, b % 5
                assert abs(ra - rb) + abs(ca - cb) == 1  # grid-adjacent
            else:
                q = g.qubits[0]
                assert g.name in ("T", "SqrtX", "SqrtY")
                if q not in prev:
                    assert g.name == "T"
                else:
                    assert prev[q] != g.name  # no repeat
                prev[q] = g.name
    assert W.to_text(W.supremacy(4, 3, 10, seed=3)) == W.to_text(W.supremacy(4, 3, 10, seed=3))
    assert W.to_text(W.supremacy(4, 3, 10, seed=3)) != W.to_text(W.supremacy(4, 3, 10, seed=4))


def test_moments_disjoint():
    for c in (W.supremacy(5, 5, 12), W.multiplier(4), W.random_circuit(8, 100, 1), W.qft(7)):
        for m in c.moments:
            qs = [q for g in m for q in g.all_qubits()]
            assert len(qs) == len(set(qs))


def test_inverse_structure():
    c = W.random_circuit(5, 30, 2)
    inv = W.inverse(c)
    assert W.gate_count(inv) == 30
    assert W.to_text(W.inverse(inv)).splitlines()[2:] == W.to_text(c).splitlines()[2:]


def test_random_state_normalised():
    psi = W.random_state(10, 0)
    assert abs(np.sum(np.abs(psi) ** 2) - 1) < 1e-12
    assert np.array_equal(psi, W.random_state(10, 0))


# ------------------------------------------------------------------ width sweep
def test_remove_random_qubit_examples():
    rng = W.circuits.Xoshiro256ss(1)
    c = W.Circuit(2, [[W.GateSpec("CNOT", (0, 1))]])
    r = W.remove_random_qubit(c, rng)
    assert r.n == 1 and W.gate_count(r) == 0 and r.depth == 0
    c = W.Circuit(3, [[W.GateSpec("H", (0,)), W.GateSpec("H", (1,)), W.GateSpec("H", (2,))]])
    for seed in range(20):
        r = W.remove_random_qubit(c, W.circuits.Xoshiro256ss(seed))
        assert r.n == 2 and [g.qubits for g in r.gates] == [(0,), (1,)]
    big = W.supremacy(5, 4, 8, seed=0)
    r = W.remove_random_qubit(big, W.circuits.Xoshiro256ss(3))
    assert r.n == 19 and W.gate_count(r) < W.gate_count(big)


def test_width_sweep_properties():
    base = W.multiplier(3)  # 13 qubits
    sweep = W.width_sweep(base, 9, seed=5)
    assert [c.n for c in sweep] == [12, 11, 10, 9]
    prev = base
    for c in sweep:
        # nested gate sets under the recorded renumbering
        r = c.meta["removed"][-1]
        back = lambda q: q if q < r else q + 1  # noqa: E731
        prev_set = {(g.name, g.qubits) for g in prev.gates}
        assert all((g.name, tuple(back(q) for q in g.qubits)) in prev_set for g in c.gates)
        for g in c.gates:
            assert max(g.all_qubits()) < c.n
        prev = c
    assert [W.to_text(c) for c in sweep] == [W.to_text(c) for c in W.width_sweep(base, 9, seed=5)]
    with pytest.raises(ValueError):
        W.width_sweep(base, 13, seed=0)
    assert len(W.width_sweep(W.supremacy(5, 1, 2), 4, seed=0)) == 1


def test_family_at_width():
    for n in (13, 19, 25, 28):
        assert W.family_at_width("supremacy", n).n == n
    # the standard grids the paper names are chosen for their own widths, so the sweep
    # takes them unchanged (golden shapes, not only widths)
    for row in GOLDEN["supremacy_width"]:
        assert W.supremacy_grid(row["width"]) == (row["rows"], row["cols"]), row["cite"]
        c = W.family_at_width("supremacy", row["width"], depth=4)
        assert c.meta.get("removed") is None and c.meta["rows"] == row["rows"] and c.meta["cols"] == row["cols"]
    # P:63's example: a 19-qubit circuit comes from the 20-qubit one (5x4) minus one qubit
    assert W.supremacy_grid(19) == (5, 4)
    assert W.family_at_width("supremacy", 19, depth=4).meta["removed"] and len(
        W.family_at_width("supremacy", 19, depth=4).meta["removed"]) == 1
    for n in range(4, 40):
        r, c = W.supremacy_grid(n)
        assert r * c >= n and c <= r <= 2 * c
    for n in (13, 14, 16, 17, 21):
        c = W.family_at_width("multiplier", n)
        assert c.n == n
    assert W.gate_count(W.family_at_width("multiplier", 17)) == W.gate_count(W.multiplier(4))
