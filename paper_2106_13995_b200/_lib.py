"""ctypes binding of libsv.so (include/sv.h).  Argument marshalling only: every step of the
path runs in the library's kernels.  There is no CPU fallback: if libsv.so is missing or
fails to load, importing this module raises."""

from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libsv.so")

SV_C64, SV_C128 = 1, 2
SV_KERNEL_AUTO, SV_KERNEL_PER_GATE, SV_KERNEL_DENSE = 0, 1, 2
STATUS = {0: "SV_OK", 1: "SV_ERR_ARG", 2: "SV_ERR_RANGE", 3: "SV_ERR_RESOURCE", 4: "SV_ERR_PARSE",
          5: "SV_ERR_CUDA", 6: "SV_ERR_NCCL", 7: "SV_ERR_STATE"}


class SvError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class RunOpts(ctypes.Structure):
    _fields_ = [("fuse", ctypes.c_int), ("tile_qubits", ctypes.c_int), ("max_fused_k", ctypes.c_int),
                ("force_kernel", ctypes.c_int), ("check_unitary", ctypes.c_int), ("use_graph", ctypes.c_int),
                ("profile", ctypes.c_int), ("exchange", ctypes.c_int)]


ALLGATHER_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p)
BARRIER_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p)


class Control(ctypes.Structure):
    """sv_control: host control plane of a sharded state (all-gather + barrier callbacks)."""
    _fields_ = [("user", ctypes.c_void_p), ("allgather", ALLGATHER_FN), ("barrier", BARRIER_FN)]


class RunStats(ctypes.Structure):
    _fields_ = [("gates", ctypes.c_uint64), ("passes", ctypes.c_uint64), ("stages", ctypes.c_uint64),
                ("swaps", ctypes.c_uint64), ("launches", ctypes.c_uint64), ("hbm_bytes", ctypes.c_uint64),
                ("nvlink_bytes", ctypes.c_uint64), ("plan_ms", ctypes.c_double)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2106_13995_b200.build` "
                          "(there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    vp, cp, i, u64 = ctypes.c_void_p, ctypes.c_char_p, ctypes.c_int, ctypes.c_uint64
    ip = ctypes.POINTER(ctypes.c_int)
    dp = ctypes.POINTER(ctypes.c_double)
    sig = {
        "sv_memory_estimate": (u64, [i, i]),
        "sv_create": (i, [i, i, vp, ctypes.POINTER(vp)]),
        "sv_wrap": (i, [i, i, vp, vp, ctypes.POINTER(vp)]),
        "sv_nccl_unique_id": (i, [vp]),
        "sv_create_sharded": (i, [i, i, vp, i, i, vp, ctypes.POINTER(vp)]),
        "sv_create_virtual_sharded": (i, [i, i, i, vp, ctypes.POINTER(vp)]),
        "sv_create_sharded_ex": (i, [i, i, vp, ctypes.POINTER(Control), i, i, vp, vp, ctypes.POINTER(vp)]),
        "sv_destroy": (i, [vp]),
        "sv_init_zero": (i, [vp]),
        "sv_init_basis": (i, [vp, u64]),
        "sv_init_uniform": (i, [vp]),
        "sv_set_amplitudes": (i, [vp, u64, u64, vp]),
        "sv_apply_gate": (i, [vp, dp, i, ip, ip, i]),
        "sv_plan_compile": (i, [cp, i, ctypes.POINTER(RunOpts), ctypes.POINTER(vp)]),
        "sv_plan_info": (i, [vp, ip, ctypes.POINTER(u64), ctypes.POINTER(u64), ctypes.POINTER(u64)]),
        "sv_plan_qubit_map": (i, [vp, ip]),
        "sv_plan_destroy": (i, [vp]),
        "sv_plan_source": (i, [vp, i, ctypes.c_char_p, ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t)]),
        "sv_plan_apply": (i, [vp, vp, ctypes.POINTER(RunStats)]),
        "sv_plan_pass_times": (i, [vp, ctypes.POINTER(ctypes.c_float), i, ip]),
        "sv_plan_shard_info": (i, [vp, i, ctypes.POINTER(u64), ctypes.POINTER(u64), ctypes.POINTER(u64)]),
        "sv_apply_circuit": (i, [vp, cp, ctypes.POINTER(RunOpts), ctypes.POINTER(RunStats)]),
        "sv_amplitudes": (i, [vp, u64, u64, vp]),
        "sv_probabilities": (i, [vp, ip, i, dp]),
        "sv_norm": (i, [vp, dp]),
        "sv_sync": (i, [vp]),
        "sv_info": (i, [vp, ip, ip, ip, ip, ip]),
        "sv_device_ptr": (i, [vp, ctypes.POINTER(vp), ctypes.POINTER(u64)]),
        "sv_stream": (i, [vp, ctypes.POINTER(vp)]),
        "sv_qubit_map": (i, [vp, ip]),
        "sv_last_error": (cp, []),
        "sv_version": (cp, []),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    return L


lib = _load()
EXPORTED = ["sv_memory_estimate", "sv_create", "sv_wrap", "sv_nccl_unique_id", "sv_create_sharded",
            "sv_create_sharded_ex",
            "sv_create_virtual_sharded", "sv_destroy", "sv_init_zero", "sv_init_basis", "sv_init_uniform",
            "sv_set_amplitudes", "sv_apply_gate", "sv_plan_compile", "sv_plan_info", "sv_plan_qubit_map", "sv_plan_source",
            "sv_plan_destroy", "sv_plan_pass_times", "sv_plan_shard_info",
            "sv_plan_apply", "sv_apply_circuit", "sv_amplitudes", "sv_probabilities", "sv_norm", "sv_sync",
            "sv_info", "sv_device_ptr", "sv_stream", "sv_qubit_map", "sv_last_error", "sv_version"]


def check(status: int) -> None:
    if status != 0:
        raise SvError(status, lib.sv_last_error().decode(errors="replace"))
