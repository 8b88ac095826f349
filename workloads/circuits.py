"""Circuit generators and the IR text writer (inputs only; no simulation arithmetic).

IR text format (extended per SURVEY 8(c) R15):

    # comment
    qubits: <n>
    family: <tag>
    meta.<key>: <value>
    <moment>            one moment per line, gates separated by ';'

    gate   := NAME q[,q...]                      named gate, controls first, target last
            | U t0[,t1...] : re,im,re,im,...      2^k x 2^k matrix, row-major; row/col bit j <-> t_j (R2)
            | CU c0[,c1...] | t0[,t1...] : ...    controlled U: applies U when every control is 1
    NAME   := X Y Z H S T Sdg Tdg SqrtX SqrtY SqrtXdg SqrtYdg CZ CNOT Toffoli SWAP

Qubit q is bit q of the basis index (little-endian).
"""

from __future__ import annotations

import dataclasses
from typing import List, Optional, Sequence, Tuple

import numpy as np

SELF_INVERSE = {"X", "Y", "Z", "H", "CZ", "CNOT", "Toffoli", "SWAP"}
INVERSE_NAME = {"S": "Sdg", "Sdg": "S", "T": "Tdg", "Tdg": "T",
                "SqrtX": "SqrtXdg", "SqrtXdg": "SqrtX",
                "SqrtY": "SqrtYdg", "SqrtYdg": "SqrtY"}
ARITY = {"X": 1, "Y": 1, "Z": 1, "H": 1, "S": 1, "T": 1, "Sdg": 1, "Tdg": 1,
         "SqrtX": 1, "SqrtY": 1, "SqrtXdg": 1, "SqrtYdg": 1,
         "CZ": 2, "CNOT": 2, "SWAP": 2, "Toffoli": 3}


@dataclasses.dataclass(frozen=True)
class GateSpec:
    name: str                     # named kind, "U" or "CU"
    qubits: Tuple[int, ...]       # named: controls first, target last; U/CU: targets
    controls: Tuple[int, ...] = ()  # CU only
    matrix: Optional[Tuple[complex, ...]] = None  # U/CU: row-major 2^k x 2^k

    def all_qubits(self) -> Tuple[int, ...]:
        return tuple(self.controls) + tuple(self.qubits)


@dataclasses.dataclass
class Circuit:
    n: int
    moments: List[List[GateSpec]]
    family: str = "custom"
    meta: dict = dataclasses.field(default_factory=dict)

    @property
    def gates(self) -> List[GateSpec]:
        return [g for m in self.moments for g in m]

    @property
    def depth(self) -> int:
        return len(self.moments)


def gate_count(c: Circuit) -> int:
    return sum(len(m) for m in c.moments)


# ---------------------------------------------------------------- PRNG
class Xoshiro256ss:
    """xoshiro256** seeded by SplitMix64; documented, seedable."""

    M = (1 << 64) - 1

    def __init__(self, seed: int):
        x = seed & self.M
        s = []
        for _ in range(4):
            x = (x + 0x9E3779B97F4A7C15) & self.M
            z = x
            z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & self.M
            z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & self.M
            s.append(z ^ (z >> 31))
        self.s = s

    @staticmethod
    def _rotl(x, k):
        return ((x << k) | (x >> (64 - k))) & Xoshiro256ss.M

    def next(self) -> int:
        s = self.s
        result = (self._rotl((s[1] * 5) & self.M, 7) * 9) & self.M
        t = (s[1] << 17) & self.M
        s[2] ^= s[0]
        s[3] ^= s[1]
        s[1] ^= s[2]
        s[0] ^= s[3]
        s[2] ^= t
        s[3] = self._rotl(s[3], 45)
        return result

    def below(self, k: int) -> int:
        """Uniform integer in [0, k) from the top 32 bits (k small; bias < 2^-29)."""
        return ((self.next() >> 32) * k) >> 32


# ---------------------------------------------------------------- supremacy (App. C)
def _cz_pattern(rows: int, cols: int, t: int, n: Optional[int] = None) -> List[Tuple[int, int]]:
    """CZ layer pat[t mod 8]: H(0,0), H(1,1), V(0,0), V(1,1), H(0,1), H(1,0), V(0,1), V(1,0).

    H(s,u) = {(r,c)-(r,c+1) : c = s, r = u (mod 2)};  V(s,u) = {(r,c)-(r+1,c) : r = s, c = u (mod 2)}.
    With n < rows*cols only the first n sites (row-major) exist (partial last row).
    """
    n = rows * cols if n is None else n
    pats = [("H", 0, 0), ("H", 1, 1), ("V", 0, 0), ("V", 1, 1),
            ("H", 0, 1), ("H", 1, 0), ("V", 0, 1), ("V", 1, 0)]
    kind, s, u = pats[t % 8]
    pairs = []
    for r in range(rows):
        for c in range(cols):
            q = r * cols + c
            if kind == "H" and c % 2 == s and r % 2 == u and c + 1 < cols and q + 1 < n:
                pairs.append((q, q + 1))
            if kind == "V" and r % 2 == s and c % 2 == u and r + 1 < rows and q + cols < n:
                pairs.append((q, q + cols))
    return pairs


def supremacy(rows: int, cols: int, depth: int, seed: int = 0, n: Optional[int] = None) -> Circuit:
    """Supremacy-style grid circuit (reading R6).

    Moment 0: H on every qubit.  Cycle t: CZ layer pat[t mod 8], then a single-qubit
    layer on every qubit not in that CZ layer: first gate T, afterwards uniform over
    {SqrtX, SqrtY, T} minus the qubit's previous gate.  `depth` counts cycles.
    n (default rows*cols) keeps only the first n sites of the grid (partial last row), used
    for the 2^30-amplitudes-per-GPU weak-scaling widths 31..33.
    """
    n = rows * cols if n is None else n
    assert 2 <= n <= rows * cols
    rng = Xoshiro256ss(seed)
    moments: List[List[GateSpec]] = [[GateSpec("H", (q,)) for q in range(n)]]
    prev: List[Optional[str]] = [None] * n
    for t in range(depth):
        pairs = _cz_pattern(rows, cols, t, n)
        moments.append([GateSpec("CZ", p) for p in pairs])
        busy = {q for p in pairs for q in p}
        layer = []
        for q in range(n):
            if q in busy:
                continue
            if prev[q] is None:
                g = "T"
            else:
                choices = [x for x in ("SqrtX", "SqrtY", "T") if x != prev[q]]
                g = choices[rng.below(len(choices))]
            prev[q] = g
            layer.append(GateSpec(g, (q,)))
        moments.append(layer)
    return Circuit(n, moments, "supremacy",
                   {"rows": rows, "cols": cols, "cycles": depth, "seed": seed})


# ---------------------------------------------------------------- multiplier (App. B)
def _asap(n: int, gates: Sequence[GateSpec]) -> List[List[GateSpec]]:
    """Pack an ordered gate list into moments (earliest moment after every gate it shares a qubit with)."""
    level = [0] * n
    moments: List[List[GateSpec]] = []
    for g in gates:
        qs = g.all_qubits()
        d = max(level[q] for q in qs)
        if d == len(moments):
            moments.append([])
        moments[d].append(g)
        for q in qs:
            level[q] = d + 1
    return moments


def multiplier_gates(na: int, nb: int) -> List[GateSpec]:
    """Controlled Cuccaro shift-and-add multiplier (reading R7).

    A = 0..na-1, B = na..na+nb-1, P = na+nb..2(na+nb)-1, ancilla = 2(na+nb).
    For each bit i of B: B_i-controlled add of A into P[i..i+na-1], carry into P[i+na].
    """
    A = list(range(na))
    B = list(range(na, na + nb))
    P = list(range(na + nb, 2 * (na + nb)))
    anc = 2 * (na + nb)
    gates: List[GateSpec] = []
    cx = lambda c, t: gates.append(GateSpec("CNOT", (c, t)))  # noqa: E731
    ccx = lambda a, b, t: gates.append(GateSpec("Toffoli", (a, b, t)))  # noqa: E731
    for i in range(nb):
        c = [anc] + A[:-1]
        z = P[i + na]
        for j in range(na):  # MAJ chain
            cx(A[j], P[i + j])
            cx(A[j], c[j])
            ccx(c[j], P[i + j], A[j])
        ccx(B[i], A[na - 1], z)  # carry-out
        for j in reversed(range(na)):  # controlled UMA chain
            ccx(c[j], P[i + j], A[j])
            cx(A[j], c[j])
            cx(A[j], P[i + j])
            ccx(B[i], A[j], P[i + j])
            ccx(B[i], c[j], P[i + j])
    return gates


def multiplier(na: int, nb: Optional[int] = None) -> Circuit:
    """Reversible multiplier |a>|b>|0>|0> -> |a>|b>|a*b>|0>, width 2(na+nb)+1 (4n+1 when square)."""
    nb = na if nb is None else nb
    n = 2 * (na + nb) + 1
    return Circuit(n, _asap(n, multiplier_gates(na, nb)), "multiplier",
                   {"operand_bits_a": na, "operand_bits_b": nb})


def basis_prep(c: Circuit, bits: int) -> Circuit:
    """Prepend X gates preparing basis state |bits> from |0...0> (SPEC design decision S:316)."""
    xs = [GateSpec("X", (q,)) for q in range(c.n) if (bits >> q) & 1]
    moments = ([xs] if xs else []) + [list(m) for m in c.moments]
    return Circuit(c.n, moments, c.family, dict(c.meta, prep=bits))


# ---------------------------------------------------------------- QFT (closed-form pin)
def _cphase(theta: float) -> Tuple[complex, ...]:
    ph = complex(np.cos(theta), np.sin(theta))
    return (1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1, 0, 0, 0, 0, ph)


def qft(n: int) -> Circuit:
    """Little-endian QFT: for t = n-1..0: H(t); for s = t-1..0: CP(pi/2^(t-s)) on (s,t);
    then SWAP(j, n-1-j).  QFT|k> = 2^(-n/2) sum_j e^{+2 pi i jk/2^n} |j> (SURVEY 8(c) pins)."""
    gates: List[GateSpec] = []
    for t in range(n - 1, -1, -1):
        gates.append(GateSpec("H", (t,)))
        for s in range(t - 1, -1, -1):
            gates.append(GateSpec("U", (s, t), (), _cphase(np.pi / 2 ** (t - s))))
    for j in range(n // 2):
        gates.append(GateSpec("SWAP", (j, n - 1 - j)))
    return Circuit(n, _asap(n, gates), "qft", {})


# ---------------------------------------------------------------- random circuits
def random_unitary(k: int, rng: np.random.Generator) -> np.ndarray:
    d = 1 << k
    z = (rng.standard_normal((d, d)) + 1j * rng.standard_normal((d, d))) / np.sqrt(2)
    q, r = np.linalg.qr(z)
    ph = np.diag(r) / np.abs(np.diag(r))
    return q * ph


def random_circuit(n: int, ngates: int, seed: int, kinds: Optional[Sequence[str]] = None,
                   max_k: int = 3, max_controls: int = 2) -> Circuit:
    """Random circuit over the full gate set: named gates, dense U (k<=max_k), diagonal U,
    permutation U, and CU with up to max_controls controls.  Gates in file order, one per
    moment when they overlap (ASAP packing)."""
    rng = np.random.default_rng(seed)
    names = list(kinds) if kinds else (
        ["X", "Y", "Z", "H", "S", "T", "Sdg", "Tdg", "SqrtX", "SqrtY", "SqrtXdg", "SqrtYdg",
         "CZ", "CNOT", "SWAP", "Toffoli", "U", "Udiag", "Uperm", "CU"])
    gates: List[GateSpec] = []
    while len(gates) < ngates:
        kind = names[rng.integers(len(names))]
        if kind in ARITY:
            a = ARITY[kind]
            if a > n:
                continue
            qs = tuple(int(x) for x in rng.choice(n, a, replace=False))
            gates.append(GateSpec(kind, qs))
            continue
        k = int(rng.integers(1, min(max_k, n) + 1))
        nc = int(rng.integers(1, max_controls + 1)) if kind == "CU" else 0
        if k + nc > n:
            continue
        qs = [int(x) for x in rng.choice(n, k + nc, replace=False)]
        ctrl, tgt = tuple(qs[:nc]), tuple(qs[nc:])
        d = 1 << k
        if kind == "Udiag":
            m = np.diag(np.exp(1j * rng.uniform(0, 2 * np.pi, d)))
        elif kind == "Uperm":
            m = np.eye(d)[rng.permutation(d)].astype(complex)
        else:
            m = random_unitary(k, rng)
        gates.append(GateSpec("CU" if nc else "U", tgt, ctrl, tuple(complex(x) for x in m.reshape(-1))))
    return Circuit(n, _asap(n, gates), "custom", {"seed": seed})


# ---------------------------------------------------------------- transforms
def _inverse_gate(g: GateSpec) -> GateSpec:
    if g.name in SELF_INVERSE:
        return g
    if g.name in INVERSE_NAME:
        return GateSpec(INVERSE_NAME[g.name], g.qubits)
    d = 1 << len(g.qubits)
    m = np.array(g.matrix, dtype=complex).reshape(d, d)
    return GateSpec(g.name, g.qubits, g.controls, tuple(complex(x) for x in m.conj().T.reshape(-1)))


def inverse(c: Circuit) -> Circuit:
    """C^dagger: reversed moment order, each gate replaced by its inverse (mirror)."""
    return Circuit(c.n, [[_inverse_gate(g) for g in reversed(m)] for m in reversed(c.moments)],
                   c.family + "-inverse", dict(c.meta))


def concat(a: Circuit, b: Circuit) -> Circuit:
    assert a.n == b.n
    return Circuit(a.n, [list(m) for m in a.moments] + [list(m) for m in b.moments],
                   a.family + "+" + b.family, dict(a.meta))


# ---------------------------------------------------------------- width sweep (f3)
def remove_random_qubit(c: Circuit, rng: Xoshiro256ss) -> Circuit:
    """SPEC S:281-289 / P:63: pick a qubit uniformly, delete every gate that touches it,
    renumber the remaining qubits in order, drop empty moments, record the removed index."""
    if c.n < 2:
        raise ValueError("cannot remove a qubit from a 1-qubit circuit")
    r = rng.below(c.n)

    def remap(q):
        return q if q < r else q - 1

    moments = []
    for m in c.moments:
        kept = []
        for g in m:
            if r in g.all_qubits():
                continue
            kept.append(GateSpec(g.name, tuple(remap(q) for q in g.qubits), tuple(remap(q) for q in g.controls),
                                 g.matrix))
        if kept:
            moments.append(kept)
    removed = list(c.meta.get("removed", [])) + [r]
    return Circuit(c.n - 1, moments, c.family, dict(c.meta, removed=removed))


def width_sweep(base: Circuit, min_width: int, seed: int) -> List[Circuit]:
    """SPEC S:291-299 / P:63: circuits of widths base.n-1 down to min_width, each obtained
    from the previous one by one random qubit removal (deterministic for a seed)."""
    if min_width >= base.n:
        raise ValueError("min_width must be below the base width")
    rng = Xoshiro256ss(seed)
    out, cur = [], base
    while cur.n > min_width:
        cur = remove_random_qubit(cur, rng)
        out.append(cur)
    return out


def supremacy_grid(n: int):
    """The standard supremacy grid a width-n circuit is taken from: the smallest
    near-square grid rows x cols >= n, rows >= cols, rows <= 2*cols (the paper ran square
    n x n grids and 7 x 4; "next largest circuit"); ties on the area go to the
    squarer grid.  25 -> 5x5, 28 -> 7x4, 36 -> 6x6, 30 -> 6x5, 19 -> 5x4 (reading in DESIGN)."""
    best = None
    for cols in range(1, 64):
        for rows in range(cols, 2 * cols + 1):
            if rows * cols < n:
                continue
            key = (rows * cols, rows - cols)
            if best is None or key < best[0]:
                best = (key, rows, cols)
    return best[1], best[2]


def family_at_width(family: str, n: int, seed: int = 0, depth: int = 20) -> Circuit:
    """The paper's method for non-standard widths: build the next larger standard circuit
    and remove random qubits.  Supremacy: the near-square grid of supremacy_grid(n);
    multiplier: width 4k+1."""
    if family == "supremacy":
        rows, cols = supremacy_grid(n)
        c = supremacy(rows, cols, depth, seed)
    elif family == "multiplier":
        k = 1
        while 4 * k + 1 < n:
            k += 1
        c = multiplier(k)
    else:
        raise ValueError(family)
    if c.n == n:
        return c
    return width_sweep(c, n, seed)[-1]


# ---------------------------------------------------------------- writer
def _fmt(x: float) -> str:
    return repr(float(x))


def _gate_text(g: GateSpec) -> str:
    if g.name in ARITY:
        return f"{g.name} " + ",".join(str(q) for q in g.qubits)
    nums = ",".join(f"{_fmt(z.real)},{_fmt(z.imag)}" for z in g.matrix)
    tg = ",".join(str(q) for q in g.qubits)
    if g.name == "CU":
        return f"CU {','.join(str(q) for q in g.controls)}|{tg} : {nums}"
    return f"U {tg} : {nums}"


def to_text(c: Circuit) -> str:
    lines = [f"qubits: {c.n}", f"family: {c.family}"]
    for k, v in c.meta.items():
        lines.append(f"meta.{k}: {v}")
    for m in c.moments:
        if m:
            lines.append("; ".join(_gate_text(g) for g in m))
    return "\n".join(lines) + "\n"
