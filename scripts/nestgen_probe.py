"""Launch list of one timed-out NESTGEN conv candidate (run under ncu)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
from conftest import load_population
from paper_2205_13603_b200.runner import B200Runner
hdr, pop = load_population("conv2d")
progs = [p["program"] for p in pop]
r = B200Runner(dtype="bf16", min_repeats=1, max_repeats=1, target_ms=0.001, timeout_ms=float(sys.argv[1]))
r.set_workload(hdr["e0"])
plans = r.plan_programs(progs)
i = next(k for k, p in enumerate(plans) if p["family"] == "nestgen")
import torch
torch.cuda.profiler.start()
res = r.measure_programs([progs[i]])
torch.cuda.profiler.stop()
print(res)
