"""The real cross-process sharded path on ONE GPU.

Several processes share cuda:0, each a rank of a sharded state created with a host control
plane (torch.distributed over gloo: all-gather + barrier callbacks; NCCL refuses two ranks
on one device).  Everything else is the multi-GPU product path: every rank maps every other
rank's buffer pair through CUDA IPC (cudaIpcGetMemHandle / cudaIpcOpenMemHandle, exchanged by
the all-gather), the pass before a global<->local exchange stores straight into the peers'
second buffers, the barrier orders those stores, the ranks flip buffers, readouts
canonicalise with pairwise peer pushes, marginals all-gather.  Each rank's slice is compared
with the fp64 oracle at indices [r 2^L, (r+1) 2^L) (SURVEY 8(c) comparison step 3).
"""

import os
import socket
import traceback

import numpy as np
import pytest
import torch.multiprocessing as mp

import oracle
import workloads as W
from tests.parity import assert_close

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q, job):
    try:
        import torch
        import torch.distributed as dist
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        import paper_2106_13995_b200 as P
        out = job(P, rank, world)
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok", out))
    except Exception:
        q.put((rank, "err", traceback.format_exc()))


def run_ranks(world, job, timeout=600):
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, job)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    try:
        for _ in range(world):
            rank, status, out = q.get(timeout=timeout)
            assert status == "ok", f"rank {rank} failed:\n{out}"
            res[rank] = out
    finally:
        for p in procs:
            p.join(timeout=60)
            if p.is_alive():
                p.kill()
    return [res[r] for r in range(world)]


# ---------------------------------------------------------------- jobs (module level: picklable)
def _job_circuit(P, rank, world, text=None, n=None, dtype=None, exchange=0, psi0=None, subset=None):
    with P.StateVector.sharded(n, dtype, control="host") as sv:
        if psi0 is not None:
            sv.set_amplitudes(psi0)
        st = sv.apply_circuit(text, exchange=exchange)
        L = 1 << sv.n_local
        amps = sv.amplitudes(rank * L, L)  # this rank's part of the logical range
        probs = sv.probabilities(subset) if subset is not None else None
        nrm = sv.norm()
        return {"amps": amps, "stats": st, "map": sv.qubit_map(), "probs": probs, "norm": nrm}


class Job:
    """Picklable closure over keyword arguments."""

    def __init__(self, fn, **kw):
        self.fn, self.kw = fn, kw

    def __call__(self, P, rank, world):
        return self.fn(P, rank, world, **self.kw)


def gather(res):
    return np.concatenate([r["amps"] for r in res])


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("dtype", ["c128", "c64"])
def test_ipc_sharded_supremacy_vs_oracle(world, dtype):
    c = W.supremacy(4, 4, 12, seed=world)
    text = W.to_text(c)
    ref = oracle.simulate(text)
    sub = [0, 15, 7, 14]  # global (top) and local qubits in the marginal
    res = run_ranks(world, Job(_job_circuit, text=text, n=16, dtype=dtype, subset=sub))
    for r in res:
        assert r["stats"]["swaps"] >= 1  # the exchange ran across processes
        assert r["map"] == list(range(16))  # readout canonicalised (peer pushes)
        assert abs(r["norm"] - 1.0) < 1e-5
        np.testing.assert_array_equal(r["probs"], res[0]["probs"])  # same value on every rank
    assert_close(gather(res), ref, dtype, W.gate_count(c))
    np.testing.assert_allclose(res[0]["probs"], oracle.probabilities(ref, sub), atol=1e-6 if dtype == "c64" else 1e-12)


def test_ipc_sharded_8_ranks():
    c = W.supremacy(4, 4, 10, seed=8)
    text = W.to_text(c)
    res = run_ranks(8, Job(_job_circuit, text=text, n=16, dtype="c128"))
    assert all(r["stats"]["swaps"] >= 1 for r in res)
    assert_close(gather(res), oracle.simulate(text), "c128", W.gate_count(c))


@pytest.mark.parametrize("seed", range(3))
def test_ipc_fused_and_copy_exchange_bit_identical(seed):
    """exchange=0 (remote stores fused into the pass) and exchange=1 (peer-copy kernel after
    the pass) move the same amplitudes to the same places: bit-identical states."""
    n = 13
    c = W.random_circuit(n, 150, 700 + seed, max_k=3, max_controls=2)
    text = W.to_text(c)
    psi0 = W.random_state(n, seed)
    fused = run_ranks(2, Job(_job_circuit, text=text, n=n, dtype="c128", psi0=psi0, exchange=0))
    copy = run_ranks(2, Job(_job_circuit, text=text, n=n, dtype="c128", psi0=psi0, exchange=1))
    np.testing.assert_array_equal(gather(fused), gather(copy))
    assert_close(gather(fused), oracle.simulate(text, psi0), "c128", W.gate_count(c))


def test_ipc_multiplier_bit_exact():
    c = W.multiplier(3)  # 13 qubits: the product register and the ancilla are the top qubits
    n = c.n
    a, b = 5, 6
    k = a | (b << 3)
    text = W.to_text(c)
    psi0 = np.zeros(1 << n, np.complex128)
    psi0[k] = 1.0
    ref = oracle.simulate(text, psi0)
    res = run_ranks(4, Job(_job_circuit, text=text, n=n, dtype="c64", psi0=psi0.astype(np.complex64)))
    got = gather(res)
    assert np.array_equal(got.astype(np.complex128), ref)  # R10: == at every index
    assert int(np.flatnonzero(got)[0]) == int(np.flatnonzero(ref)[0])


def _job_repeat(P, rank, world, text=None, n=None):
    """The same circuit three times on one state: the buffer pair flips back and forth."""
    with P.StateVector.sharded(n, "c128", control="host") as sv:
        for _ in range(3):
            sv.apply_circuit(text)
        L = 1 << sv.n_local
        return {"amps": sv.amplitudes(rank * L, L)}


def test_ipc_repeated_applies_flip_buffers():
    c = W.supremacy(4, 3, 8, seed=3)
    text = W.to_text(c)
    ref = oracle.simulate(text)
    for _ in range(2):
        ref = oracle.simulate(text, ref)
    res = run_ranks(2, Job(_job_repeat, text=text, n=12))
    assert_close(gather(res), ref, "c128", 3 * W.gate_count(c))


def _job_borrowed(P, rank, world, text=None, n=None):
    import torch
    L = 1 << (n - (world.bit_length() - 1))
    buf = torch.zeros(L, dtype=torch.complex128, device="cuda")
    with P.StateVector.sharded(n, "c128", control="host", buffer=buf) as sv:
        sv.apply_circuit(text)
        sv.sync()
        direct = buf.cpu().numpy().copy()  # the caller's tensor, read without the library
        return {"amps": direct, "map": sv.qubit_map()}


def test_ipc_borrowed_shard_buffer_holds_logical_order():
    c = W.supremacy(4, 4, 12, seed=1)
    text = W.to_text(c)
    res = run_ranks(2, Job(_job_borrowed, text=text, n=16))
    assert all(r["map"] == list(range(16)) for r in res)
    assert_close(gather(res), oracle.simulate(text), "c128", W.gate_count(c))


def _job_gather(P, rank, world, text=None, n=None):
    with P.StateVector.sharded(n, "c128", control="host") as sv:
        sv.apply_circuit(text)
        full = sv.gather_amplitudes(root=0)
        return {"full": full}


def test_ipc_gather_amplitudes_to_rank0():
    c = W.supremacy(4, 4, 8, seed=4)
    text = W.to_text(c)
    res = run_ranks(4, Job(_job_gather, text=text, n=16))
    assert res[0]["full"] is not None and all(r["full"] is None for r in res[1:])
    assert_close(res[0]["full"], oracle.simulate(text), "c128", W.gate_count(c))


def _job_mismatch(P, rank, world, texts=None):
    from paper_2106_13995_b200._lib import SvError
    with P.StateVector.sharded(12, "c128", control="host") as sv:
        try:
            sv.apply_circuit(texts[rank])
        except SvError as e:
            return {"status": e.status, "msg": str(e)}
        return {"status": 0, "msg": ""}


def test_ipc_ranks_with_different_plans_fail_before_launch():
    """Every rank compares plan signatures before the first launch: a rank that was given
    another circuit makes every rank fail with SV_ERR_STATE instead of hanging or mixing."""
    t0 = W.to_text(W.supremacy(4, 3, 6, seed=0))
    t1 = W.to_text(W.supremacy(4, 3, 6, seed=1))
    res = run_ranks(2, Job(_job_mismatch, texts=[t0, t1]))
    for r in res:
        assert r["status"] == 7, r  # SV_ERR_STATE
        assert "differs between ranks" in r["msg"]


def test_bench_multirank_host_control_plane():
    """bench.py's N > 1 path (torchrun, one process per rank, sharded state, max over ranks,
    one JSON line from rank 0) with two ranks sharing this GPU through the host control plane
    (--control host): weak scaling, 2^24 amplitudes per rank."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.join(root, "bench.py"),
           "--gpus", "2", "--control", "host", "--workload", "weak", "--qubits", "24", "--steps", "3",
           "--warmup", "3"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=root)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["n_qubits"] == 25 and d["value"] > 0
    assert d["config"]["swaps_per_step"] >= 1 and d["scaling"] == "weak"
    assert d["e2e"]["value"] > 0
