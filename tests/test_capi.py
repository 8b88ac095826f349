"""CPU-side checks of the boundary: libsv.so builds, loads and exports every symbol that
include/sv.h declares; host-only calls behave (no compute calls without a GPU)."""

import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    txt = open(os.path.join(ROOT, "include", "sv.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(sv_[a-z_0-9]+)\s*\(", txt)))


def test_header_declares_the_north_star_calls():
    syms = declared_symbols()
    for s in ["sv_create", "sv_apply_gate", "sv_apply_circuit", "sv_probabilities", "sv_amplitudes"]:
        assert s in syms


def test_library_exports_every_declared_symbol():
    from paper_2106_13995_b200 import _lib
    lib = ctypes.CDLL(_lib.LIB_PATH)
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    assert sorted(_lib.EXPORTED) == declared_symbols()


def test_kernels_are_sm100a():
    """The shared library carries sm_100a SASS (cuobjdump lists the arch)."""
    import shutil
    import subprocess
    from paper_2106_13995_b200 import _lib
    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(tool):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([tool, "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_host_only_calls():
    import paper_2106_13995_b200 as P
    assert P.memory_estimate(42, "c128") == 70368744177664  # P:38 "42-qubit ... 64TB"
    assert P.memory_estimate(30, "c64") == 8 * 2 ** 30
    assert P.memory_estimate(61, "c128") == 2 ** 64 - 1     # saturates (R20)
    from paper_2106_13995_b200._lib import lib
    assert lib.sv_version().decode().startswith("svb")


def test_plan_compile_parse_errors():
    """IR parse errors name the 1-based line without touching a GPU."""
    import paper_2106_13995_b200 as P
    with pytest.raises(P.SvError, match="line 3"):
        P.Plan("qubits: 3\nH 0\nFOO 1\n")
    with pytest.raises(P.SvError, match="line 2"):
        P.Plan("qubits: 3\nCZ 1,1\n")
    with pytest.raises(P.SvError, match="SV_ERR_PARSE"):
        P.Plan("H 0\n")
    # a second header after gates were range-checked against the first: rejected
    with pytest.raises(P.SvError, match="line 4.*repeated"):
        P.Plan("qubits: 20\nH 19\nX 18\nqubits: 2\n")
    with pytest.raises(P.SvError, match="repeated"):
        P.Plan("qubits: 3\nqubits: 3\nH 0\n")
    # unused ABI slot must be zero
    from paper_2106_13995_b200._lib import RunOpts, lib
    import ctypes
    h = ctypes.c_void_p()
    o = RunOpts(1, 0, 3, 0, 0, 0, 0, 0)
    assert lib.sv_plan_compile(b"qubits: 2\nH 0\n", 1, ctypes.byref(o), ctypes.byref(h)) == 1  # SV_ERR_ARG
    p = P.Plan("qubits: 4\nH 0; CNOT 0,1\nU 2 : 1,0,0,0,0,0,1,0\n")
    assert p.info()["gates"] == 3 and p.info()["n"] == 4


def test_sharded_ex_argument_errors_before_any_cuda_call():
    """sv_create_sharded_ex validates its arguments before touching CUDA or NCCL."""
    from paper_2106_13995_b200._lib import Control, lib
    h = ctypes.c_void_p()
    # neither a unique id nor a control plane
    assert lib.sv_create_sharded_ex(10, 1, None, None, 2, 0, None, None, ctypes.byref(h)) == 1
    assert b"exactly one" in lib.sv_last_error()
    # a control plane without callbacks
    c = Control()
    assert lib.sv_create_sharded_ex(10, 1, None, ctypes.byref(c), 2, 0, None, None, ctypes.byref(h)) == 1
    # world not a power of two / too large, rank out of range
    uid = (ctypes.c_uint8 * 128)()
    for world, rank in ((3, 0), (16, 0), (2, 2)):
        assert lib.sv_create_sharded_ex(10, 1, ctypes.cast(uid, ctypes.c_void_p), None, world, rank, None, None,
                                        ctypes.byref(h)) == 1


def test_check_unitary_option():
    """sv_run_opts.check_unitary rejects a non-unitary matrix at plan time (SV_ERR_ARG with the
    line); unchecked plans accept it (unitarity is not checked by default)."""
    import paper_2106_13995_b200 as P
    bad = "qubits: 2\nH 1\nU 0 : 1,0,1,0,0,0,1,0\n"
    with pytest.raises(P.SvError, match="line 3.*not unitary"):
        P.Plan(bad, "c64", check_unitary=True)
    P.Plan(bad, "c64")
    P.Plan("qubits: 2\nH 0\nU 1 : 0,0,1,0,1,0,0,0\n", "c128", check_unitary=True)
