"""Launch the best candidate of one family of a population once more (no
deadline), for an ncu capture: python scripts/profile_family.py conv2d simt_affine"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
from conftest import load_population
from paper_2205_13603_b200.runner import B200Runner
name, fam = sys.argv[1], sys.argv[2]
hdr, pop = load_population(name)
dtype = "f32" if name == "gmm512" else "bf16"
progs = [p["program"] for p in pop]
r = B200Runner(dtype=dtype, min_repeats=1, max_repeats=1, target_ms=0.001, timeout_ms=5.0, timeout_factor=10.0)
r.set_workload(hdr["e0"])
plans = r.plan_programs(progs)
idx = [i for i, p in enumerate(plans) if p["family"] == fam and p["status"] == "OK"]
res = r.measure_programs([progs[i] for i in idx])
best = min((x["latency_ns"], i) for x, i in zip(res, idx) if x["status"] == "OK")[1]
r2 = B200Runner(dtype=dtype, min_repeats=1, max_repeats=1, target_ms=0.001, timeout_ms=1e7)
r2.set_workload(hdr["e0"])
import torch  # cudaProfilerStart/Stop: capture only this launch (ncu --profile-from-start off)
torch.cuda.profiler.start()
res2 = r2.measure_programs([progs[best]])
torch.cuda.profiler.stop()
print("profiling", fam, plans[best]["cfg"], res2)
