"""Host-side logic of the N > 1 path, on CPU: the sharded planner's dry run (SURVEY 8(e),
App. D model: ~1 swap for 36q d20 at P = 2/4/8) and the torch.distributed plumbing (NCCL
unique-id broadcast, max-over-ranks timing) with the gloo backend at world_size 2."""

import os
import socket

import pytest
import torch.multiprocessing as mp

import workloads as W


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2106_13995_b200.dist import broadcast_unique_id, max_over_ranks
    uid = bytes((i * 7 + 3) % 256 for i in range(128)) if rank == 0 else bytes(128)
    got = broadcast_unique_id(uid)
    mx = max_over_ranks([float(rank), 10.0 - rank, 2.5])
    q.put((rank, got, mx))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_uid_broadcast_and_max():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    expect = bytes((i * 7 + 3) % 256 for i in range(128))
    for rank, got, mx in res:
        assert got == expect
        assert mx == [1.0, 10.0, 2.5]


def _ctl_worker(rank, world, port, q):
    import ctypes

    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2106_13995_b200.dist import host_control
    c = host_control()
    # call the C function pointers exactly as libsv.so does (sv_control)
    msg = (ctypes.c_ubyte * 5)(*[rank * 10 + i for i in range(5)])
    out = (ctypes.c_ubyte * (5 * world))()
    rc = c.allgather(None, ctypes.cast(msg, ctypes.c_void_p), 5, ctypes.cast(out, ctypes.c_void_p))
    rb = c.barrier(None)
    q.put((rank, rc, rb, bytes(out)))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_host_control_plane_callbacks(world):
    """The sv_control callbacks (torch.distributed over gloo) gather in rank order and
    return 0; this is the control plane the one-GPU multi-process sharded tests use."""
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_ctl_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    expect = bytes(r * 10 + i for r in range(world) for i in range(5))
    for rank, rc, rb, out in res:
        assert rc == 0 and rb == 0
        assert out == expect


@pytest.mark.parametrize("world", [2, 4, 8])
def test_shard_plan_36q_supremacy(world):
    """Config 5: 36q c64 supremacy d20 sharded over P GPUs needs one exchange step."""
    import paper_2106_13995_b200 as P
    plan = P.Plan(W.to_text(W.supremacy(6, 6, 20, seed=0)), "c64")
    info = plan.shard_info(world)
    assert info["swaps"] == 1 and info["batches"] == 2
    assert 10 <= info["passes"] <= 24


def test_shard_plan_scaling_widths():
    import paper_2106_13995_b200 as P
    for n, world in [(31, 2), (32, 4), (33, 8), (35, 2)]:
        rows = (n + 4) // 5
        plan = P.Plan(W.to_text(W.supremacy(rows, 5, 20, seed=0, n=n)), "c64")
        info = plan.shard_info(world)
        assert 1 <= info["swaps"] <= 3, (n, world, info)


def test_shard_plan_random_and_multiplier():
    import paper_2106_13995_b200 as P
    for text in (W.to_text(W.random_circuit(14, 300, 3, max_k=3)), W.to_text(W.multiplier(4))):
        for world in (2, 4):
            info = P.Plan(text, "c128").shard_info(world)
            assert info["batches"] == info["swaps"] + 1
    with pytest.raises(P.SvError):
        P.Plan("qubits: 4\nH 0\n").shard_info(3)


def test_planner_pass_counts_regression():
    """Host planner regression pins (measured plans of DESIGN.md 6.1 / 7): the 30 q supremacy
    d20 circuit in 7 passes for both dtypes (relabelling + rollout), and the weak-scaling
    shards with relabelled batches (31 q / P = 2: 8 passes per shard, 33 q / P = 8: 10)."""
    import paper_2106_13995_b200 as P
    text = W.to_text(W.supremacy(6, 5, 20, seed=0))
    assert P.Plan(text, "c64").info()["passes"] <= 7
    assert P.Plan(text, "c128").info()["passes"] <= 7
    for n, world, most in [(31, 2, 8), (33, 8, 10)]:
        t = W.to_text(W.supremacy((n + 4) // 5, 5, 20, seed=0, n=n))
        info = P.Plan(t, "c64").shard_info(world)
        assert info["swaps"] == 1 and info["passes"] <= most, (n, world, info)
