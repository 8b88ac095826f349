"""Summaries of ncu CSV exports: launch lists and --set full details (used for profiles/)."""
import csv
import sys
from collections import defaultdict


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hdr]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    out = defaultdict(dict)
    for r in rows[hdr + 1:]:
        out[(int(r[0]), r[ki][:40])][r[mi]] = float(r[vi].replace(",", ""))
    tot = 0
    for k, v in sorted(out.items()):
        t = v["gpu__time_duration.sum"] / 1e6
        tot += t
        b = v.get("dram__bytes_read.sum", 0) + v.get("dram__bytes_write.sum", 0)
        print(f"{k[0]:3d} {k[1]:40s} {t:8.3f} ms  {b / 1e9:6.2f} GB  {b / t / 1e6 if t else 0:7.0f} GB/s")
    print(f"total {tot:.3f} ms")


def details(path, sections=("GPU Speed Of Light Throughput", "Memory Workload Analysis", "Warp State Statistics",
                            "Occupancy", "Compute Workload Analysis", "Instruction Statistics",
                            "Scheduler Statistics")):
    rows = list(csv.reader(open(path)))
    h = rows[0]
    si, mi, ui, vi = h.index("Section Name"), h.index("Metric Name"), h.index("Metric Unit"), h.index("Metric Value")
    for r in rows[1:]:
        if r[si] in sections and r[mi]:
            print(f"{r[si][:26]:26s} | {r[mi]} = {r[vi]} {r[ui]}")


def stalls(path):
    rows = list(csv.reader(open(path)))
    d = dict(zip(rows[0], rows[2] if len(rows) > 2 else rows[1]))
    st = []
    for k, v in d.items():
        if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued"):
            try:
                st.append((float(v.replace(",", "")), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    tot = sum(x for x, _ in st) or 1
    for x, k in sorted(st, reverse=True)[:12]:
        print(f"stall {k:28s} {100 * x / tot:5.1f} %")
    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
              "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
              "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__inst_executed.sum"):
        if k in d:
            print(f"{k} = {d[k]}")


if __name__ == "__main__":
    mode, path = sys.argv[1], sys.argv[2]
    {"launches": launches, "details": details, "stalls": stalls}[mode](path)
