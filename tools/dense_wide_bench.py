"""Single dense k = 3..5 gates at 30 qubits through sv_apply_gate (dense-k kernels): device ms
(CUDA events, median of 5) and the fractions of the HBM and FP floors."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2106_13995_b200 as P  # noqa: E402

n = 30
peak = float(json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"]) if os.path.exists("MEASURED_PEAKS.json") else 6550.0
for dtype in ("c64", "c128"):
    b = 8 if dtype == "c64" else 16
    fp = 148 * (128 if dtype == "c64" else 64) * 1.965e9  # FP lane-ops/s (DESIGN 6)
    with P.StateVector(n, dtype) as sv:
        sv.init_uniform()
        stream = torch.cuda.ExternalStream(sv.stream_ptr())
        for k, tg in ((3, [1, 12, n - 3]), (4, [0, 6, 13, n - 2]), (5, [2, 5, 11, 19, n - 1])):
            r = np.random.default_rng(k)
            d = 1 << k
            U, _ = np.linalg.qr(r.normal(size=(d, d)) + 1j * r.normal(size=(d, d)))
            for _ in range(2):
                sv.apply_gate(U, tg)
            sv.sync()
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(5)]
            for e0, e1 in ev:
                e0.record(stream)
                sv.apply_gate(U, tg)
                e1.record(stream)
            sv.sync()
            ms = sorted(e0.elapsed_time(e1) for e0, e1 in ev)[2]
            t_hbm = 2 * (1 << n) * b / (peak * 1e9) * 1e3
            t_fp = (1 << n) * 4 * d / fp * 1e3  # 4 * 2^k FMA lane-ops per amplitude (2^k complex MACs)
            print(json.dumps({"dtype": dtype, "k": k, "ms": round(ms, 3), "hbm_floor_ms": round(t_hbm, 3),
                              "fp_floor_ms": round(t_fp, 3), "floor_frac": round(max(t_hbm, t_fp) / ms, 3)}), flush=True)
