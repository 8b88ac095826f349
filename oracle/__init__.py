"""ctypes wrapper of the CPU oracle (oracle/sv_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / ``--impl reference`` legs.  Never imported by paper_2106_13995_b200/.
See sv_oracle.c's header for what is computed and which passages it follows.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "sv_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile liboracle.so: gcc -O2 -ffp-contract=off -fopenmp (reading R18)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=gnu11", "-ffp-contract=off", "-fno-fast-math",
                               "-fopenmp", "-fPIC", "-shared", _SRC, "-o", _LIB, "-lm"])
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        dp = ctypes.POINTER(ctypes.c_double)
        ip = ctypes.POINTER(ctypes.c_int)
        up = ctypes.POINTER(ctypes.c_uint64)
        L.or_apply_gate.argtypes = [ctypes.c_int, dp, dp, ctypes.c_int, ip, ip, ctypes.c_int, ctypes.c_int]
        L.or_circuit_info.argtypes = [ctypes.c_char_p, ip, ip, ctypes.c_char_p, ctypes.c_int]
        L.or_run.argtypes = [ctypes.c_char_p, dp, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                             ctypes.c_int, ctypes.c_char_p, ctypes.c_int]
        L.or_init_zero.argtypes = [ctypes.c_int, dp]
        L.or_init_uniform.argtypes = [ctypes.c_int, dp]
        L.or_memory_estimate.argtypes = [ctypes.c_int, ctypes.c_int]
        L.or_memory_estimate.restype = ctypes.c_uint64
        L.or_norm.argtypes = [ctypes.c_int, dp]
        L.or_norm.restype = ctypes.c_double
        L.or_probabilities.argtypes = [ctypes.c_int, dp, ip, ctypes.c_int, dp]
        L.or_classical_map.argtypes = [ctypes.c_char_p, up, up, ctypes.c_uint64, ctypes.c_char_p, ctypes.c_int]
        L.or_classical_map_range.argtypes = [ctypes.c_char_p, ctypes.c_uint64, ctypes.c_uint64, up,
                                             ctypes.c_char_p, ctypes.c_int]
        L.or_max_threads.restype = ctypes.c_int
        _lib = L
    return _lib


class OracleError(RuntimeError):
    pass


def _dp(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _ip(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int))


def circuit_info(text: str):
    n, g = ctypes.c_int(), ctypes.c_int()
    err = ctypes.create_string_buffer(256)
    if lib().or_circuit_info(text.encode(), ctypes.byref(n), ctypes.byref(g), err, 256):
        raise OracleError(err.value.decode())
    return n.value, g.value


def zero_state(n: int) -> np.ndarray:
    psi = np.empty(1 << n, dtype=np.complex128)
    lib().or_init_zero(n, _dp(psi))
    return psi


def uniform_state(n: int) -> np.ndarray:
    psi = np.empty(1 << n, dtype=np.complex128)
    lib().or_init_uniform(n, _dp(psi))
    return psi


def run(text: str, psi: np.ndarray, first: int = 0, count: int = -1, nthreads: int = 0) -> np.ndarray:
    """Apply gates [first, first+count) of `text` to psi (complex128, modified in place)."""
    assert psi.dtype == np.complex128 and psi.flags.c_contiguous
    n = int(psi.size).bit_length() - 1
    err = ctypes.create_string_buffer(256)
    if lib().or_run(text.encode(), _dp(psi), n, first, count, nthreads, err, 256):
        raise OracleError(err.value.decode())
    return psi


def simulate(text: str, psi_in: np.ndarray = None, nthreads: int = 0) -> np.ndarray:
    n, _ = circuit_info(text)
    psi = zero_state(n) if psi_in is None else np.array(psi_in, dtype=np.complex128, copy=True)
    return run(text, psi, nthreads=nthreads)


def apply_gate(psi: np.ndarray, U: np.ndarray, targets, controls=(), nthreads: int = 0) -> np.ndarray:
    n = int(psi.size).bit_length() - 1
    U = np.ascontiguousarray(U, dtype=np.complex128)
    t = np.array(targets, dtype=np.int32)
    c = np.array(controls if len(controls) else [0], dtype=np.int32)
    rc = lib().or_apply_gate(n, _dp(psi), _dp(U), len(targets), _ip(t), _ip(c), len(controls), nthreads)
    if rc:
        raise OracleError(f"or_apply_gate failed ({rc})")
    return psi


def norm(psi: np.ndarray) -> float:
    n = int(psi.size).bit_length() - 1
    return lib().or_norm(n, _dp(np.ascontiguousarray(psi, dtype=np.complex128)))


def probabilities(psi: np.ndarray, qubits) -> np.ndarray:
    n = int(psi.size).bit_length() - 1
    q = np.array(list(qubits) or [0], dtype=np.int32)
    out = np.zeros(1 << len(qubits), dtype=np.float64)
    if lib().or_probabilities(n, _dp(np.ascontiguousarray(psi)), _ip(q), len(qubits), _dp(out)):
        raise OracleError("bad qubit list")
    return out


def memory_estimate(n: int, bytes_per_amp: int = 16) -> int:
    return int(lib().or_memory_estimate(n, bytes_per_amp))


def classical_map(text: str, inputs: np.ndarray) -> np.ndarray:
    inp = np.ascontiguousarray(inputs, dtype=np.uint64)
    out = np.empty_like(inp)
    err = ctypes.create_string_buffer(256)
    up = ctypes.POINTER(ctypes.c_uint64)
    if lib().or_classical_map(text.encode(), inp.ctypes.data_as(up), out.ctypes.data_as(up),
                              inp.size, err, 256):
        raise OracleError(err.value.decode())
    return out


def classical_map_range(text: str, first: int, count: int, out: np.ndarray = None) -> np.ndarray:
    """f(i) for i in [first, first+count) (bit-sliced, X/SWAP-type gates with controls; first and
    count multiples of 64).  SURVEY 8(c) comparison step 5."""
    if out is None:
        out = np.empty(count, dtype=np.uint64)
    assert out.dtype == np.uint64 and out.size >= count and out.flags.c_contiguous
    err = ctypes.create_string_buffer(256)
    if lib().or_classical_map_range(text.encode(), int(first), int(count),
                                    out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), err, 256):
        raise OracleError(err.value.decode())
    return out


def max_threads() -> int:
    return int(lib().or_max_threads())
