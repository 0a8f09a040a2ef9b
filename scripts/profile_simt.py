"""Launch one SIMT candidate of a population (for ncu): --cfg prefix."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
from conftest import load_population
from paper_2205_13603_b200.runner import B200Runner
name, want = sys.argv[1], [int(x) for x in sys.argv[2].split(",")]
hdr, pop = load_population(name)
r = B200Runner(dtype="f32" if name == "gmm512" else "bf16", min_repeats=2, max_repeats=2, target_ms=0.001,
               timeout_ms=1e7)  # no deadline: ncu replays stretch wall time
r.set_workload(hdr["e0"])
progs = [p["program"] for p in pop]
plans = r.plan_programs(progs)
i = next(i for i, p in enumerate(plans) if p["status"] == "OK" and p["cfg"][:len(want)] == want)
print(plans[i]["family"], plans[i]["cfg"], r.measure_programs([progs[i]]))
