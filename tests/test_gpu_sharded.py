"""Sharded execution: the state split over P shards by its top log2(P) qubits,
global<->local qubit swaps, rank-constant folding of controls and diagonals on global qubits,
and readout after the qubit map is made canonical.  On one GPU this runs the same planner,
qubit map and swap schedule through sv_create_virtual_sharded (shards are slices of one
allocation; the exchange is device-to-device copies), compared with the oracle."""

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


def run_virtual(P, text, n, world, dtype, psi0=None, **opts):
    with P.StateVector.virtual_sharded(n, world, dtype) as sv:
        if psi0 is not None:
            sv.set_amplitudes(psi0)
        st = sv.apply_circuit(text, **opts)
        amps = sv.amplitudes()
        qmap = sv.qubit_map()
        return amps, st, qmap


@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("dtype", ["c128", "c64"])
def test_supremacy_sharded_matches_oracle(P, world, dtype):
    c = W.supremacy(4, 4, 12, seed=world)
    text = W.to_text(c)
    ref = oracle.simulate(text)
    got, st, qmap = run_virtual(P, text, 16, world, dtype)
    assert st["swaps"] >= 1  # dense gates on the top qubits forced at least one exchange
    assert qmap == list(range(16))  # readout canonicalised the map
    assert_close(got, ref, dtype, W.gate_count(c))


@pytest.mark.parametrize("seed", range(6))
@pytest.mark.parametrize("world", [2, 4])
def test_random_circuits_sharded(P, seed, world):
    n = 12
    c = W.random_circuit(n, 120, 50 + seed, max_k=4, max_controls=2)
    text = W.to_text(c)
    psi0 = W.random_state(n, seed)
    ref = oracle.simulate(text, psi0)
    for opts in ({}, {"fuse": False}):
        got, st, _ = run_virtual(P, text, n, world, "c128", psi0, **opts)
        assert_close(got, ref, "c128", W.gate_count(c))


def test_multiplier_sharded_bit_exact(P):
    c = W.multiplier(3)  # 13 qubits, top qubits hold the product register and the ancilla
    text = W.to_text(c)
    for a, b in [(5, 3), (7, 7), (6, 0)]:
        x = a | (b << 3)
        psi0 = np.zeros(1 << c.n, complex)
        psi0[x] = 1
        ref = oracle.simulate(text, psi0)
        got, st, _ = run_virtual(P, text, c.n, 4, "c128", psi0)
        assert np.array_equal(got, ref), (a, b)


def test_sharded_probabilities_and_norm(P):
    n, world = 14, 4
    c = W.supremacy(7, 2, 10, seed=3)
    text = W.to_text(c)
    ref = oracle.simulate(text)
    with P.StateVector.virtual_sharded(n, world, "c128") as sv:
        sv.apply_circuit(text)
        # before canonicalisation (map may be permuted): marginals are map-aware
        for qs in ([13], [0, 12, 13], [5, 2], list(range(n))):
            assert np.max(np.abs(sv.probabilities(qs) - oracle.probabilities(ref, qs))) <= 1e-12
        assert abs(sv.norm() - 1) <= 1e-12


def test_sharded_apply_gate_on_global_qubit(P):
    n, world = 10, 4
    rng = np.random.default_rng(4)
    psi0 = W.random_state(n, 4)
    U = W.circuits.random_unitary(2, rng)
    with P.StateVector.virtual_sharded(n, world, "c128") as sv:
        sv.set_amplitudes(psi0)
        sv.apply_gate(U, [9, 2], [8])     # dense target and control on global qubits
        sv.apply_gate(np.diag([1, 1j]), [9])  # diagonal on a global qubit: rank constant
        got = sv.amplitudes()
    ref = oracle.apply_gate(psi0.copy(), U, [9, 2], [8])
    ref = oracle.apply_gate(ref, np.diag([1, 1j]), [9])
    assert np.max(np.abs(got - ref)) <= 1e-13
