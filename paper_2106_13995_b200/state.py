"""Thin Python layer over the C-ABI: StateVector, Plan, simulate().

Marshalling only (arguments in, buffers out); the state lives in HBM and every gate,
initialisation and readout runs in libsv.so's kernels.  PyTorch is used only for the
device, streams and torch.distributed (NCCL unique-id broadcast for sharded states).
"""

from __future__ import annotations

import ctypes
from typing import Iterable, Optional, Sequence

import numpy as np

from ._lib import RunOpts, RunStats, SV_C128, SV_C64, check, lib

_DT = {"c64": SV_C64, "complex64": SV_C64, SV_C64: SV_C64,
       "c128": SV_C128, "complex128": SV_C128, SV_C128: SV_C128}
_NP = {SV_C64: np.complex64, SV_C128: np.complex128}


def _dtype(d) -> int:
    if d in _DT:
        return _DT[d]
    if d in (np.complex64,):
        return SV_C64
    if d in (np.complex128,):
        return SV_C128
    raise ValueError(f"unknown dtype {d!r}")


def make_opts(fuse: bool = True, tile_qubits: int = 0, force_kernel: int = 0, check_unitary: bool = False,
              use_graph: bool = False, profile: bool = False, exchange: int = 0) -> RunOpts:
    return RunOpts(int(fuse), int(tile_qubits), 0, int(force_kernel), int(check_unitary), int(use_graph),
                   int(profile), int(exchange))


def _stream_ptr(stream) -> Optional[int]:
    if stream is None:
        return None
    return int(getattr(stream, "cuda_stream", stream))


class Plan:
    """A compiled circuit (parse + classify + fuse + plan), reusable across states/runs."""

    def __init__(self, text: str, dtype="c64", **opts):
        self.dtype = _dtype(dtype)
        self._h = ctypes.c_void_p()
        self._opts = make_opts(**opts)
        check(lib.sv_plan_compile(text.encode(), self.dtype, ctypes.byref(self._opts), ctypes.byref(self._h)))

    def info(self):
        n = ctypes.c_int()
        g, p, s = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
        check(lib.sv_plan_info(self._h, ctypes.byref(n), ctypes.byref(g), ctypes.byref(p), ctypes.byref(s)))
        return {"n": n.value, "gates": g.value, "passes": p.value, "stages": s.value}

    def qubit_map(self):
        """Logical -> physical qubit map the single-GPU schedule leaves behind."""
        n = self.info()["n"]
        out = (ctypes.c_int * n)()
        check(lib.sv_plan_qubit_map(self._h, out))
        return list(out)

    def shard_info(self, world: int) -> dict:
        """Host-only dry run of the sharded schedule over `world` GPUs (no GPU needed)."""
        s, b, p = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
        check(lib.sv_plan_shard_info(self._h, int(world), ctypes.byref(s), ctypes.byref(b), ctypes.byref(p)))
        return {"swaps": s.value, "batches": b.value, "passes": p.value}

    def pass_times(self):
        """Per-pass device ms of the last apply (plan compiled with profile=True)."""
        n = ctypes.c_int()
        check(lib.sv_plan_pass_times(self._h, None, 0, ctypes.byref(n)))
        buf = (ctypes.c_float * max(1, n.value))()
        check(lib.sv_plan_pass_times(self._h, buf, n.value, ctypes.byref(n)))
        return list(buf)[: n.value]

    def source(self, i: int) -> str:
        """Generated CUDA source of tile pass i (single-GPU schedule)."""
        ln = ctypes.c_size_t()
        check(lib.sv_plan_source(self._h, int(i), None, 0, ctypes.byref(ln)))
        buf = ctypes.create_string_buffer(ln.value + 1)
        check(lib.sv_plan_source(self._h, int(i), buf, ln.value + 1, ctypes.byref(ln)))
        return buf.value.decode()

    def close(self):
        if self._h:
            lib.sv_plan_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class StateVector:
    """2^n complex amplitudes in HBM (optionally sharded over GPUs by the top qubits)."""

    def __init__(self, n: int, dtype="c64", stream=None, _handle=None):
        self.dtype = _dtype(dtype)
        self._h = ctypes.c_void_p()
        if _handle is not None:
            self._h = _handle
        else:
            check(lib.sv_create(int(n), self.dtype, _stream_ptr(stream), ctypes.byref(self._h)))
        self._refresh()

    def _refresh(self):
        n, nl, w, r, dt = (ctypes.c_int() for _ in range(5))
        check(lib.sv_info(self._h, *(ctypes.byref(x) for x in (n, nl, w, r, dt))))
        self.n, self.n_local, self.world, self.rank = n.value, nl.value, w.value, r.value

    # ---------------------------------------------------------------- constructors
    @classmethod
    def wrap(cls, tensor, n: int, stream=None) -> "StateVector":
        """Borrow a contiguous complex64/complex128 CUDA tensor of 2^n elements."""
        import torch
        assert tensor.is_cuda and tensor.is_contiguous() and tensor.numel() == (1 << n)
        dt = SV_C64 if tensor.dtype == torch.complex64 else SV_C128
        h = ctypes.c_void_p()
        check(lib.sv_wrap(int(n), dt, ctypes.c_void_p(tensor.data_ptr()), _stream_ptr(stream), ctypes.byref(h)))
        sv = cls(n, dt, _handle=h)
        sv._borrowed = tensor
        return sv

    @classmethod
    def virtual_sharded(cls, n: int, world: int, dtype="c64", stream=None) -> "StateVector":
        h = ctypes.c_void_p()
        check(lib.sv_create_virtual_sharded(int(n), _dtype(dtype), int(world), _stream_ptr(stream),
                                            ctypes.byref(h)))
        return cls(n, dtype, _handle=h)

    @classmethod
    def sharded(cls, n: int, dtype="c64", group=None, stream=None, control: str = "nccl",
                buffer=None) -> "StateVector":
        """Collective: one process per rank, each on its current CUDA device.

        control="nccl": the library's own NCCL communicator; torch.distributed broadcasts the
        unique id.  control="host": torch.distributed itself is the control plane (all-gather
        + barrier callbacks, any backend incl. gloo) and every exchange goes through CUDA IPC
        peer memory -- several ranks may then share one GPU.  buffer: optional contiguous
        complex CUDA tensor of 2^(n - log2 world) elements to borrow as the local shard."""
        import torch.distributed as dist

        from .dist import broadcast_unique_id, host_control
        world, rank = dist.get_world_size(group), dist.get_rank(group)
        ptr = None
        if buffer is not None:
            assert buffer.is_cuda and buffer.is_contiguous()
            ptr = ctypes.c_void_p(buffer.data_ptr())
        h = ctypes.c_void_p()
        keep = None
        if control == "nccl":
            uid = (ctypes.c_uint8 * 128)()
            if rank == 0:
                check(lib.sv_nccl_unique_id(ctypes.cast(uid, ctypes.c_void_p)))
            raw = broadcast_unique_id(bytes(uid), group)
            ctypes.memmove(uid, raw, 128)
            check(lib.sv_create_sharded_ex(int(n), _dtype(dtype), ctypes.cast(uid, ctypes.c_void_p), None, world,
                                           rank, ptr, _stream_ptr(stream), ctypes.byref(h)))
        elif control == "host":
            keep = host_control(group)
            check(lib.sv_create_sharded_ex(int(n), _dtype(dtype), None, ctypes.byref(keep), world, rank, ptr,
                                           _stream_ptr(stream), ctypes.byref(h)))
        else:
            raise ValueError(f"control must be 'nccl' or 'host', not {control!r}")
        sv = cls(n, dtype, _handle=h)
        sv._control = keep  # the callbacks must outlive the handle
        sv._borrowed = buffer
        return sv

    # ---------------------------------------------------------------- init
    def init_zero(self):
        check(lib.sv_init_zero(self._h))
        return self

    def init_basis(self, k: int):
        check(lib.sv_init_basis(self._h, int(k)))
        return self

    def init_uniform(self):
        check(lib.sv_init_uniform(self._h))
        return self

    def set_amplitudes(self, values: np.ndarray, first: int = 0):
        a = np.ascontiguousarray(values, dtype=_NP[self.dtype])
        check(lib.sv_set_amplitudes(self._h, int(first), a.size, a.ctypes.data_as(ctypes.c_void_p)))
        return self

    # ---------------------------------------------------------------- apply
    def apply_gate(self, U, targets: Sequence[int], controls: Sequence[int] = ()):
        U = np.ascontiguousarray(U, dtype=np.complex128)
        k = len(targets)
        t = (ctypes.c_int * k)(*targets)
        c = (ctypes.c_int * max(1, len(controls)))(*controls) if controls else None
        check(lib.sv_apply_gate(self._h, U.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), k, t, c,
                                len(controls)))
        return self

    def apply_circuit(self, text: str, **opts) -> dict:
        o = make_opts(**opts)
        st = RunStats()
        check(lib.sv_apply_circuit(self._h, text.encode(), ctypes.byref(o), ctypes.byref(st)))
        return st.as_dict()

    def apply_plan(self, plan: Plan) -> dict:
        st = RunStats()
        check(lib.sv_plan_apply(self._h, plan._h, ctypes.byref(st)))
        return st.as_dict()

    # ---------------------------------------------------------------- readout
    def amplitudes(self, first: int = 0, count: Optional[int] = None) -> np.ndarray:
        if count is None:
            count = (1 << self.n) - first
        out = np.zeros(count, dtype=_NP[self.dtype])
        check(lib.sv_amplitudes(self._h, int(first), int(count), out.ctypes.data_as(ctypes.c_void_p)))
        return out

    def gather_amplitudes(self, root: int = 0, group=None) -> Optional[np.ndarray]:
        """Sharded states (collective): every rank reads the part of the logical index range it
        holds and `root` receives the whole 2^n vector (small n only); other
        ranks get None.  Unsharded states: all amplitudes."""
        if self.world == 1:
            return self.amplitudes()
        import torch
        import torch.distributed as dist
        L = 1 << self.n_local
        mine = self.amplitudes(self.rank * L, L)
        t = torch.from_numpy(mine.view(np.float64 if self.dtype == SV_C128 else np.float32).copy())
        backend_cuda = dist.get_backend(group) == "nccl"
        if backend_cuda:
            t = t.cuda()
        parts = [torch.empty_like(t) for _ in range(self.world)] if dist.get_rank(group) == root else None
        dist.gather(t, parts, dst=root, group=group)
        if parts is None:
            return None
        flat = torch.cat([p.cpu() for p in parts]).numpy()
        return flat.view(_NP[self.dtype])

    def probabilities(self, qubits: Iterable[int]) -> np.ndarray:
        qs = list(qubits)
        q = (ctypes.c_int * max(1, len(qs)))(*qs)
        out = np.zeros(1 << len(qs), dtype=np.float64)
        check(lib.sv_probabilities(self._h, q, len(qs), out.ctypes.data_as(ctypes.POINTER(ctypes.c_double))))
        return out

    def norm(self) -> float:
        v = ctypes.c_double()
        check(lib.sv_norm(self._h, ctypes.byref(v)))
        return v.value

    def sync(self):
        check(lib.sv_sync(self._h))

    def stream_ptr(self) -> int:
        p = ctypes.c_void_p()
        check(lib.sv_stream(self._h, ctypes.byref(p)))
        return p.value or 0

    def device_ptr(self):
        p, n = ctypes.c_void_p(), ctypes.c_uint64()
        check(lib.sv_device_ptr(self._h, ctypes.byref(p), ctypes.byref(n)))
        return p.value, n.value

    def qubit_map(self):
        out = (ctypes.c_int * self.n)()
        check(lib.sv_qubit_map(self._h, out))
        return list(out)

    def close(self):
        if self._h:
            lib.sv_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


def memory_estimate(n: int, dtype="c128") -> int:
    return int(lib.sv_memory_estimate(int(n), _dtype(dtype)))


def simulate(text: str, dtype="c64", init: str = "zero", **opts) -> np.ndarray:
    """SPEC S:542-550 bound_simulate: run a circuit from |0> (or uniform) and return all amplitudes."""
    n = None
    for line in text.splitlines():
        if line.strip().startswith("qubits:"):
            n = int(line.split(":", 1)[1])
            break
    if n is None:
        raise ValueError("IR text has no 'qubits:' header")
    with StateVector(n, dtype) as sv:
        if init == "uniform":
            sv.init_uniform()
        sv.apply_circuit(text, **opts)
        return sv.amplitudes()
