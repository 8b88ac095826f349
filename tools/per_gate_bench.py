"""Single-gate kernels at 30 qubits: one sv_apply_gate call = one pass over
the state (per-gate mode, the precompiled tile-pass kernel), device time by CUDA events on the
state's stream, after warm-up; GB/s = 2 x state bytes / time against the measured HBM peak.

python tools/per_gate_bench.py [--qubits 30] [--reps 5]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2106_13995_b200 as P  # noqa: E402
import workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--qubits", type=int, default=30)
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
n = a.qubits
try:
    peak = float(json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                             "MEASURED_PEAKS.json")))["hbm_gbs"])
except Exception:
    peak = 6650.0
h = 2 ** -0.5
H = np.array([[h, h], [h, -h]])
X = np.array([[0, 1], [1, 0]], complex)
T = np.diag([1, np.exp(1j * np.pi / 4)])
Z = np.diag([1, -1]).astype(complex)
rng = np.random.default_rng(0)
q, _ = np.linalg.qr(rng.normal(size=(4, 4)) + 1j * rng.normal(size=(4, 4)))
U2 = q
def haar(k, seed):
    r = np.random.default_rng(seed)
    d = 1 << k
    qq, _ = np.linalg.qr(r.normal(size=(d, d)) + 1j * r.normal(size=(d, d)))
    return qq


cases = [("dense U3 q1,q12,q27", haar(3, 3), [1, 12, n - 3], []),
         ("dense U4 q0,q6,q13,q28", haar(4, 4), [0, 6, 13, n - 2], []),
         ("dense U5 q2,q5,q11,q19,q29", haar(5, 5), [2, 5, 11, 19, n - 1], []),
         ("H q0", H, [0], []), ("H q14", H, [14], []), ("H q29", H, [n - 1], []),
         ("T q7", T, [7], []), ("CZ q3,q20", Z, [20], [3]), ("CNOT q0->q29", X, [n - 1], [0]),
         ("CNOT q29->q1", X, [1], [n - 1]), ("Toffoli q2,q9->q25", X, [25], [2, 9]),
         ("dense U2 q5,q17", U2, [5, 17], [])]
for dtype in ("c64", "c128"):
    b = 8 if dtype == "c64" else 16
    with P.StateVector(n, dtype) as sv:
        sv.init_uniform()
        stream = torch.cuda.ExternalStream(sv.stream_ptr())
        for name, U, tg, ct in cases:
            for _ in range(2):
                sv.apply_gate(U, tg, ct)
            sv.sync()
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.reps)]
            for e0, e1 in ev:
                e0.record(stream)
                sv.apply_gate(U, tg, ct)
                e1.record(stream)
            sv.sync()
            ms = sorted(e0.elapsed_time(e1) for e0, e1 in ev)[a.reps // 2]
            gbs = 2 * (1 << n) * b / (ms * 1e-3) / 1e9
            row = {"dtype": dtype, "gate": name, "ms": round(ms, 3), "GB/s (2 x state)": round(gbs),
                   "frac_of_measured_peak": round(gbs / peak, 3)}
            # the same gate as a one-gate circuit through the generic dense-k kernel (ablation)
            g = W.GateSpec("CU" if ct else "U", tuple(tg), tuple(ct),
                           tuple(complex(x) for x in np.asarray(U, complex).reshape(-1)))
            text = W.to_text(W.Circuit(n, [[g]]))
            for _ in range(2):
                sv.apply_circuit(text, force_kernel=2)
            sv.sync()
            for e0, e1 in ev:
                e0.record(stream)
                sv.apply_circuit(text, force_kernel=2)
                e1.record(stream)
            sv.sync()
            ms2 = sorted(e0.elapsed_time(e1) for e0, e1 in ev)[a.reps // 2]
            row["dense_k_ms"] = round(ms2, 3)
            row["dense_k_frac"] = round(2 * (1 << n) * b / (ms2 * 1e-3) / 1e9 / peak, 3)
            print(json.dumps(row), flush=True)
