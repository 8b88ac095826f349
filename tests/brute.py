"""Brute-force 2^n x 2^n reference (tests only; independent of oracle/ and of the CUDA path).

Definition (SURVEY 8(c) "Brute-force definition", restating SPEC S:178-196 in index form):
for a gate with targets T, controls C and matrix U (row/col bit j <-> T[j]),
    Full[i][i'] = U[r(i)][r(i')] * [i, i' agree outside T]   if every control bit of i is 1
                = delta(i, i')                                otherwise,
with r(i) = sum_j bit_{T[j]}(i) 2^j.  psi_out = Full_G ... Full_1 psi_in.
Controls are a predicate here (not a controlled-form block matrix as in the oracle), and the
gate table is built from algebraic identities rather than literals, so a slip in either
the oracle's embedding or its table fails tests/test_oracle.py.
"""

from __future__ import annotations

import numpy as np

_I2 = np.eye(2, dtype=complex)
_X = np.array([[0, 1], [1, 0]], dtype=complex)
_Z = np.diag([1, -1]).astype(complex)
_Y = 1j * _X @ _Z
_H = (_X + _Z) / np.sqrt(2)
_S = np.diag([1, 1j])
_T = np.diag([1, np.exp(1j * np.pi / 4)])
_SX = ((1 + 1j) * _I2 + (1 - 1j) * _X) / 2
_SY = ((1 + 1j) * _I2 + (1 - 1j) * _Y) / 2
_SWAP = np.eye(4, dtype=complex)[[0, 2, 1, 3]]

# name -> (number of controls, U on the target(s))
TABLE = {
    "X": (0, _X), "Y": (0, _Y), "Z": (0, _Z), "H": (0, _H),
    "S": (0, _S), "Sdg": (0, _S.conj().T), "T": (0, _T), "Tdg": (0, _T.conj().T),
    "SqrtX": (0, _SX), "SqrtXdg": (0, _SX.conj().T), "SqrtY": (0, _SY), "SqrtYdg": (0, _SY.conj().T),
    "CZ": (1, _Z), "CNOT": (1, _X), "Toffoli": (2, _X), "SWAP": (0, _SWAP),
}


def gate_parts(g):
    """GateSpec -> (U, targets, controls)."""
    if g.name in TABLE:
        nc, U = TABLE[g.name]
        return U, tuple(g.qubits[nc:]), tuple(g.qubits[:nc])
    d = 1 << len(g.qubits)
    return np.array(g.matrix, dtype=complex).reshape(d, d), tuple(g.qubits), tuple(g.controls)


def embed(n: int, U: np.ndarray, targets, controls=()) -> np.ndarray:
    N = 1 << n
    i = np.arange(N)
    r = np.zeros(N, dtype=np.int64)
    for j, t in enumerate(targets):
        r |= ((i >> t) & 1) << j
    tmask = sum(1 << t for t in targets)
    rest = i & ~tmask
    same = rest[:, None] == rest[None, :]
    ctl = np.ones(N, dtype=bool)
    for c in controls:
        ctl &= ((i >> c) & 1) == 1
    full = np.where(same, U[r[:, None], r[None, :]], 0)
    return np.where(ctl[:, None], full, np.eye(N))


def simulate(circ, psi_in=None) -> np.ndarray:
    n = circ.n
    psi = np.zeros(1 << n, dtype=complex) if psi_in is None else np.array(psi_in, dtype=complex)
    if psi_in is None:
        psi[0] = 1
    for g in circ.gates:
        U, t, c = gate_parts(g)
        psi = embed(n, U, t, c) @ psi
    return psi
