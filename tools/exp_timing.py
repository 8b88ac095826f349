import sys, os, time
sys.path.insert(0, os.getcwd())
mode = sys.argv[1]
if "torch" in mode:
    import torch
    torch.cuda.set_device(0)
import workloads as W, paper_2106_13995_b200 as P
c = W.supremacy(6, 5, 20, 0)
plan = P.Plan(W.to_text(c), "c64", profile=True)
sv = P.StateVector(30, "c64")
if "smi" in mode:
    import subprocess
    pr = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm", "--format=csv", "-lms", "100"], stdout=subprocess.DEVNULL)
for _ in range(4):
    sv.init_zero(); sv.apply_plan(plan)
t = plan.pass_times()
print(mode, "total", round(sum(t), 2), [round(x, 2) for x in t])
if "smi" in mode:
    pr.terminate()
