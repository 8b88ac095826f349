"""torch.distributed plumbing for sharded states and the multi-GPU bench (host logic only).

One process per GPU; torch.distributed carries the 128-byte NCCL unique id
(rank 0 -> all, N5) and the max-over-ranks reduction of device timings.  The state exchange
itself runs inside libsv.so (peer-memory stores over NVLink, or NCCL).  Alternatively
torch.distributed is the library's whole control plane (host_control: all-gather + barrier
callbacks of an sv_control), which works over gloo and lets several ranks share one GPU.
The helpers work with the gloo backend (CPU tensors) and the nccl backend (CUDA tensors),
so their logic is tested on CPU with world_size 2.
"""

from __future__ import annotations

from typing import List, Sequence


def _device_for(group=None):
    import torch
    import torch.distributed as dist
    return torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" \
        else torch.device("cpu")


def broadcast_unique_id(uid: bytes, group=None) -> bytes:
    """Rank 0's 128-byte NCCL unique id, on every rank (collective)."""
    import torch
    import torch.distributed as dist
    assert len(uid) == 128
    t = torch.tensor(list(uid), dtype=torch.uint8, device=_device_for(group))
    dist.broadcast(t, src=0, group=group)
    return bytes(t.cpu().tolist())


def max_over_ranks(values: Sequence[float], group=None) -> List[float]:
    """Element-wise max over ranks (device timings are reported as the max, not the mean)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor(list(values), dtype=torch.float64, device=_device_for(group))
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return [float(x) for x in t.cpu().tolist()]


def host_control(group=None):
    """An sv_control whose all-gather and barrier are torch.distributed collectives on `group`
    (called collectively by libsv.so from the thread making the sv_* call).  Keep the returned
    object alive as long as the state handle."""
    import ctypes

    import torch
    import torch.distributed as dist

    from ._lib import ALLGATHER_FN, BARRIER_FN, Control
    world = dist.get_world_size(group)
    dev = _device_for(group)

    def allgather(user, src, nbytes, dst):
        try:
            t = torch.frombuffer(bytearray(ctypes.string_at(src, nbytes)), dtype=torch.uint8).to(dev)
            outs = [torch.empty(nbytes, dtype=torch.uint8, device=dev) for _ in range(world)]
            dist.all_gather(outs, t, group=group)
            data = bytes(torch.cat(outs).cpu().numpy().tobytes())
            ctypes.memmove(dst, data, nbytes * world)
            return 0
        except Exception:  # an exception must not unwind through C
            return 1

    def barrier(user):
        try:
            dist.barrier(group=group)
            return 0
        except Exception:
            return 1

    fns = (ALLGATHER_FN(allgather), BARRIER_FN(barrier))
    c = Control(None, *fns)
    c._keep = fns  # the C function pointers live as long as these objects
    return c
