"""Per-kernel device time of a few conv2d candidates (run under ncu)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
from conftest import load_population
from paper_2205_13603_b200.runner import B200Runner
hdr, pop = load_population("conv2d")
r = B200Runner(dtype="bf16", min_repeats=1, max_repeats=1, target_ms=0.001, timeout_ms=50)
r.set_workload(hdr["e0"], seed=0)
progs = [p["program"] for p in pop]
res = r.measure_programs(progs)
ok = sorted([(x["latency_ns"], i) for i, x in enumerate(res) if x["status"] == "OK"])
print("best", [(round(l / 1e3, 1), res[i]["family"], res[i]["cfg"][:11]) for l, i in ok[:5]])
best = [progs[i] for _, i in ok[:3]]
r2 = B200Runner(dtype="bf16", min_repeats=1, max_repeats=1, target_ms=0.001, timeout_ms=50)
r2.set_workload(hdr["e0"], seed=0)
print(r2.measure_programs(best)[0]["latency_ns"])
