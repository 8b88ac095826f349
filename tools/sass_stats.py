"""Static instruction mix of every generated pass kernel (CPU only: nvcc -cubin + cuobjdump).

python tools/sass_stats.py [--workload supremacy|multiplier] [--dtype c64] [--qubits 30]
Prints per pass: stages, registers, SASS instructions per thread and per amplitude
(each thread owns 2^RB amplitudes), FP instructions per amplitude, shared-memory ops.
"""
import argparse
import collections
import os
import re
import subprocess
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402
import paper_2106_13995_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="supremacy")
ap.add_argument("--dtype", default="c64")
ap.add_argument("--qubits", type=int, default=30)
ap.add_argument("--tile", type=int, default=0)
a = ap.parse_args()
if a.workload == "supremacy":
    c = W.supremacy(6, 5, 20, 0) if a.qubits == 30 else W.supremacy((a.qubits + 4) // 5, 5, 20, 0, n=a.qubits)
elif a.workload == "qft":
    c = W.qft(a.qubits)
else:
    c = W.multiplier(8, 7)
plan = P.Plan(W.to_text(c), a.dtype, tile_qubits=a.tile)
info = plan.info()
print(info)
tot = collections.Counter()
with tempfile.TemporaryDirectory() as d:
    for i in range(info["passes"]):
        src = plan.source(i)
        if not src:
            print(i, "non-tile pass")
            continue
        hdr = src.splitlines()[0]
        rb = int(re.search(r"rb=(\d+)", hdr).group(1))
        f = os.path.join(d, f"p{i}.cu")
        open(f, "w").write(src)
        r = subprocess.run(["nvcc", "-cubin", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-Xptxas", "-v",
                            f, "-o", f + ".cubin"], capture_output=True, text=True)
        regs = re.search(r"Used (\d+) registers", r.stderr)
        sass = subprocess.run(["cuobjdump", "-sass", f + ".cubin"], capture_output=True, text=True).stdout
        ops = re.findall(r"^\s+/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9]+)", sass, re.M)
        cnt = collections.Counter(ops)
        n = len(ops)
        fp = sum(cnt[k] for k in ("FADD", "FFMA", "FMUL", "DADD", "DFMA", "DMUL", "FADD2", "FFMA2", "FMUL2"))
        R = 1 << rb
        # FP pipe cycles per warp on one SMSP (B200, tools/micro/fp_rate.cu): FADD2/FMUL2 2,
        # FFMA2 with an immediate 2 (3 with three register operands), scalar FP32 1, DADD/DMUL 2, DFMA 2.2
        pipe = (2 * (cnt["FADD2"] + cnt["FMUL2"]) + 2 * cnt["FFMA2"] + cnt["FADD"] + cnt["FFMA"] + cnt["FMUL"]
                + 2 * (cnt["DADD"] + cnt["DMUL"]) + 2.2 * cnt["DFMA"])
        tot.update(cnt)
        print(f"pass {i}: {hdr[24:]}, regs {regs.group(1) if regs else '?'}, instr/thread {n}, "
              f"instr/amp {n / R:.1f}, fp/amp {fp / R:.1f}, fp-pipe cyc/amp {pipe / R:.1f}, lds+sts {cnt['LDS'] + cnt['STS']}, "
              f"bra {cnt['BRA']}, local {cnt['LDL'] + cnt['STL']}")
