"""Stall breakdown + pipe utilisation of one ncu report (run here on the .ncu-rep)."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, v = rows[0], rows[2] if len(rows) > 2 else rows[1]
d = dict(zip(h, v))
tot = 0
st = {}
for k, x in d.items():
    if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
        try:
            st[k[len("smsp__pcsamp_warps_issue_stalled_"):]] = float(x)
        except ValueError:
            pass
tot = sum(st.values()) or 1
print("duration ms", d.get("gpu__time_duration.sum"))
for k, x in sorted(st.items(), key=lambda t: -t[1])[:10]:
    print(f"  stall {k:22s} {100 * x / tot:5.1f} %")
for k in ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
          "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
          "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active",
          "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
          "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
          "sm__warps_active.avg.pct_of_peak_sustained_active", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
          "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smsp__inst_executed.sum"):
    if k in d:
        print(f"  {k} = {d[k]}")
