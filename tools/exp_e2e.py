"""Break down the e2e step (sv_apply_circuit through the plan cache + marginal readout)."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
torch.cuda.set_device(0)
import workloads as W, paper_2106_13995_b200 as P
wl = sys.argv[1] if len(sys.argv) > 1 else "supremacy"
c = W.supremacy(6, 5, 20, 0) if wl == "supremacy" else W.multiplier(8, 7)
text = W.to_text(c)
sv = P.StateVector(c.n, "c64")
plan = P.Plan(text, "c64")
for _ in range(3):
    sv.init_zero(); sv.apply_plan(plan); sv.apply_circuit(text); sv.probabilities(range(20))
sv.sync()
def t(f, k=5):
    sv.sync(); t0 = time.perf_counter()
    for _ in range(k): f()
    sv.sync(); return (time.perf_counter() - t0) / k * 1e3
print(wl)
print("init+apply_plan ms", t(lambda: (sv.init_zero(), sv.apply_plan(plan))))
print("init+apply_circuit ms", t(lambda: (sv.init_zero(), sv.apply_circuit(text))))
print("probabilities(20) ms", t(lambda: sv.probabilities(range(20))))
print("norm ms", t(lambda: sv.norm()))
print("amplitudes 2^20 ms (canonicalises)", t(lambda: sv.amplitudes(0, 1 << 20), 1))
