"""Host-side plan shapes (no GPU): the schedule choices of plan_schedule that the bench and the
small-circuit configs depend on.  Correctness of the chosen plans is covered by the emulator
(tests/test_generator_cpu.py) and the GPU parity tests."""
import re

import pytest

import workloads as W


@pytest.fixture(scope="module")
def P():
    import paper_2106_13995_b200 as P
    return P


def _rb(plan, i):
    return int(re.search(r"rb=(\d+)", plan.source(i)).group(1))


def test_bench_plan_complex64_six_passes(P):
    # BASELINE config 3 complex64: the 128-byte-run tiles save a pass (7 -> 6)
    plan = P.Plan(W.to_text(W.supremacy(6, 5, 20, seed=0)), "c64")
    assert plan.info()["passes"] == 6
    assert all(_rb(plan, i) == 5 for i in range(6))  # no pass above the heavy threshold


def test_bench_plan_complex128(P):
    plan = P.Plan(W.to_text(W.supremacy(6, 5, 20, seed=0)), "c128")
    assert plan.info()["passes"] == 7


@pytest.mark.parametrize("dtype,rows,cols,rb", [("c128", 4, 3, 2), ("c128", 4, 4, 2), ("c64", 7, 2, 2)])
def test_small_states_take_fewer_register_bits(P, dtype, rows, cols, rb):
    # BASELINE config 1 (12 q c128) and other small states: every pass <= 64 tiles, so the
    # plan with the fewest passes and the fewest register bits per thread is kept
    c = W.supremacy(rows, cols, 10, seed=0)
    plan = P.Plan(W.to_text(c), dtype)
    for i in range(plan.info()["passes"]):
        assert _rb(plan, i) == rb


def test_large_states_keep_default_register_bits(P):
    plan = P.Plan(W.to_text(W.supremacy(6, 4, 10, seed=0)), "c128")  # 24 q: not a small state
    assert _rb(plan, 0) == 4
