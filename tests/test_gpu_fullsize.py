"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times (default
plan: fused generated passes, m = 13/12 tile qubits, 256 threads), via properties that hold at
any size or outputs the oracle computes one by one (SURVEY 8(c) comparison procedure)."""

import numpy as np
import pytest

import oracle
import workloads as W
from tests.parity import U_C64, U_C128, assert_close

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_2106_13995_b200 as P
    return P


@pytest.mark.parametrize("dtype", ["c64", "c128"])
def test_30q_supremacy_mirror(P, dtype):
    """Config 3 at full width: C then C^dagger returns |0>, norm preserved."""
    c = W.supremacy(6, 5, 20, seed=0)
    mirror = W.concat(c, W.inverse(c))
    G = W.gate_count(mirror)
    u = U_C64 if dtype == "c64" else U_C128
    with P.StateVector(30, dtype) as sv:
        st = sv.apply_plan(P.Plan(W.to_text(c), dtype))
        assert abs(sv.norm() - 1) <= 8 * W.gate_count(c) * u
        sv.apply_plan(P.Plan(W.to_text(W.inverse(c)), dtype))
        a0 = complex(sv.amplitudes(0, 1)[0])
        head = sv.amplitudes(1, 1 << 16)
        nrm = sv.norm()
    assert st["passes"] <= 16
    assert abs(a0 - 1) <= 8 * G * u
    assert np.max(np.abs(head)) <= 8 * G * u
    assert abs(nrm - 1) <= 8 * G * u


def test_24q_supremacy_d20_full_state_vs_oracle(P):
    """Same circuit family, depth and launch configuration, at a width the oracle finishes."""
    c = W.supremacy(6, 4, 20, seed=1)
    text = W.to_text(c)
    ref = oracle.simulate(text)
    for dtype in ("c64", "c128"):
        with P.StateVector(24, dtype) as sv:
            st = sv.apply_circuit(text)
            got = sv.amplitudes()
        assert st["passes"] >= 2  # several tiles per pass and several passes
        assert_close(got, ref, dtype, W.gate_count(c))


@pytest.mark.parametrize("n", [33, 34])
def test_beyond_2_32_amplitudes(P, n):
    """R22: 64-bit offsets past 2^32 amplitudes on one GPU (33q c64 = 64 GiB, 34q = 128 GiB):
    a GHZ-like state across the top qubits, closed form; then a mirror circuit returns |0>."""
    top, mid = n - 1, n - 2
    text = (f"qubits: {n}\nX {top}\nH {mid}\nCNOT {mid},0\nCNOT {mid},{n - 3}\nT {mid}\nH {top}\n")
    h = 2 ** -0.5
    with P.StateVector(n, "c64") as sv:
        sv.apply_circuit(text)
        # X(top) H(mid) CNOT CNOT T(mid) H(top): amplitudes on |top in {0,1}> x {|0>, |mid,n-3,0>}
        base1 = (1 << mid) | (1 << (n - 3)) | 1
        t = np.exp(1j * np.pi / 4)
        expect = {0: h * h, 1 << top: -h * h, base1: h * h * t, base1 | (1 << top): -h * h * t}
        for idx, val in expect.items():
            got = complex(sv.amplitudes(idx, 1)[0])
            assert abs(got - val) <= 1e-6, (idx, got, val)
        assert abs(sv.norm() - 1) <= 1e-6
        p = sv.probabilities([top, mid])
        assert np.max(np.abs(p - 0.25)) <= 1e-6
    c = W.supremacy(7, 5, 4, seed=2, n=n)
    with P.StateVector(n, "c64") as sv:
        sv.apply_circuit(W.to_text(W.concat(c, W.inverse(c))))
        assert abs(complex(sv.amplitudes(0, 1)[0]) - 1) <= 1e-4
        assert abs(sv.norm() - 1) <= 1e-4


def test_31q_multiplier_basis_exact(P):
    """Config 4 at full width (8x7 multiplier, c64): basis inputs map exactly to the oracle's
    classical image (bit-level evaluator), amplitude exactly 1, norm exactly 1 (R10)."""
    c = W.multiplier(8, 7)
    text = W.to_text(c)
    rng = np.random.default_rng(31)
    xs = [int(x) for x in rng.integers(0, 1 << 31, 6, dtype=np.int64)]
    xs += [255 | (127 << 8)]  # a = 255, b = 127, empty product register
    ys = oracle.classical_map(text, np.array(xs, dtype=np.uint64))
    plan = P.Plan(text, "c64")
    with P.StateVector(31, "c64") as sv:
        for x, y in zip(xs, ys.tolist()):
            sv.init_basis(x)
            sv.apply_plan(plan)
            assert sv.amplitudes(int(y), 1)[0] == 1 + 0j, (x, y)
            assert sv.norm() == 1.0
    a, b = 255, 127
    assert int(ys[-1]) == a | (b << 8) | ((a * b) << 15)


def _available_ram():
    try:
        return int([l for l in open("/proc/meminfo") if l.startswith("MemAvailable")][0].split()[1]) * 1024
    except Exception:
        return 0


def test_30q_bench_circuit_every_amplitude_vs_oracle(P):
    """The exact bench.py workload (config 3: 30 q supremacy d20, seed 0), launched the way
    bench.py times it (compiled plan, init_zero deferred into the first pass, fused generated
    passes), compared with the fp64 oracle amplitude by amplitude over all 2^30 indices, for
    both dtypes (streamed in chunks; bounds of reading R9)."""
    need = (16 << 30) + (2 << 30)
    if _available_ram() < need:
        pytest.skip(f"host RAM: the 30 q fp64 oracle state needs {need >> 30} GiB")
    c = W.supremacy(6, 5, 20, seed=0)
    text = W.to_text(c)
    G = W.gate_count(c)
    ref = oracle.simulate(text)  # 16 GiB complex128, all host cores
    chunk = 1 << 25
    for dtype in ("c64", "c128"):
        u = U_C64 if dtype == "c64" else U_C128
        plan = P.Plan(text, dtype)
        with P.StateVector(30, dtype) as sv:
            sv.init_zero()
            st = sv.apply_plan(plan)
            mx, l2 = 0.0, 0.0
            for first in range(0, 1 << 30, chunk):
                got = sv.amplitudes(first, chunk).astype(np.complex128)
                d = np.abs(got - ref[first:first + chunk])
                mx = max(mx, float(d.max()))
                l2 += float(np.sum(d * d))
        assert st["passes"] >= 2
        assert mx <= (1e-4 if dtype == "c64" else 1e-10), (dtype, mx)
        assert np.sqrt(l2) <= 8 * G * u, (dtype, np.sqrt(l2), 8 * G * u)
