import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
from conftest import load_population
from paper_2205_13603_b200.runner import B200Runner
hdr, pop = load_population("conv2d")
progs = [p["program"] for p in pop[:1024]]
r = B200Runner(dtype="bf16", min_repeats=3, max_repeats=50, target_ms=0.02, timeout_ms=8.8, timeout_factor=10.0,
               single_shot_factor=5.0)
r.set_workload(hdr["e0"])
plans = r.plan_programs(progs)
ng = [i for i, p in enumerate(plans) if p["family"] == "nestgen"]
tc = [i for i, p in enumerate(plans) if p["family"] == "tcgen05_conv"][:4]
for name, sel in [("ng alone", ng[:8]), ("tc+ng", tc + ng[:8]), ("full", list(range(len(progs))))]:
    res = r.measure_programs([progs[i] for i in sel])
    lat = [round(x["latency_ns"] / 1e3, 1) for x, i in zip(res, sel) if plans[i]["family"] == "nestgen"]
    print(name, "nestgen us:", lat[:8], "elapsed", round(r.elapsed_ms(), 2), r.debug_stats()["device_best_us"])
