"""Distribution of the abort latency of timed-out candidates (bench settings)."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
from conftest import load_population
from paper_2205_13603_b200.runner import B200Runner
name = sys.argv[1] if len(sys.argv) > 1 else "bert_ffn"
hdr, pop = load_population(name)
dtype = "f32" if name == "gmm512" else "bf16"
r = B200Runner(dtype=dtype, min_repeats=3, max_repeats=50, target_ms=0.02, timeout_ms=float(os.environ.get('TMO_MS', '0.9')), timeout_factor=10.0,
               timeout_floor_ms=0.05)
r.set_workload(hdr["e0"], seed=0)
progs = [p["program"] for p in pop[:1024]]
for it in range(2):
    res = r.measure_programs(progs)
to = [x for x in res if x["status"] == "TIMEOUT"]
lat = np.array([x["latency_ns"] / 1e3 for x in to])
ok = [x for x in res if x["status"] == "OK"]
best = min(x["latency_ns"] for x in ok) / 1e3
print(f"{name}: {len(to)} timeouts, best ok {best:.1f} us; abort us p10/p50/p90/max:",
      np.percentile(lat, [10, 50, 90]).round(1), lat.max().round(1))
# slowest aborts with their configs
for x in sorted(to, key=lambda x: -x["latency_ns"])[:8]:
    print(round(x["latency_ns"] / 1e3, 1), x["family"], x["cfg"])
print("elapsed ms", r.elapsed_ms(), "stats", r.debug_stats())
