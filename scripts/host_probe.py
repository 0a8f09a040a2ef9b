"""Host-side cost of one measure call (plan / phase A / phase B host ms) for a bench slice."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
from conftest import load_population
from paper_2205_13603_b200.runner import B200Runner
name = sys.argv[1] if len(sys.argv) > 1 else "bert_ffn"
hdr, pop = load_population(name)
r = B200Runner(dtype="bf16", min_repeats=3, max_repeats=50, target_ms=0.02, timeout_ms=0.9, timeout_factor=10.0,
               single_shot_factor=5.0)
r.set_workload(hdr["e0"], seed=0)
progs = [p["program"] for p in pop[:1024]]
plans = r.plan_programs(progs)
from collections import Counter
print(Counter((p["family"], p["status"]) for p in plans))
for it in range(4):
    t0 = time.perf_counter()
    res = r.measure_programs(progs)
    wall = time.perf_counter() - t0
    print(f"wall {wall*1e3:.1f} ms device {r.elapsed_ms():.1f} ms",
          {k: round(v, 2) for k, v in r.debug_stats().items()})
t0 = time.perf_counter()
for _ in range(3):
    r.plan_programs(progs)
print(f"plan only: {(time.perf_counter()-t0)/3*1e3:.1f} ms")
