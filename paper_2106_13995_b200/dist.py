"""torch.distributed plumbing for sharded states and the multi-GPU bench (host logic only).

One process per GPU; torch.distributed carries only the 128-byte NCCL unique id
(rank 0 -> all, N5) and the max-over-ranks reduction of device timings.  The state exchange
itself is NCCL inside libsv.so.  Both helpers work with the gloo backend (CPU tensors) and
the nccl backend (CUDA tensors), so their logic is tested on CPU with world_size 2.
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
