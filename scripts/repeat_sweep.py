"""Per-launch latency of the fastest schedules of a family against the number
of timed repeats in the runner's graph: a fixed per-graph cost (graph start,
first-launch effects) shows up as latency falling with the repeat count.
  python scripts/repeat_sweep.py bmm_qk tcgen05 [dtype]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from conftest import load_population  # noqa: E402
from paper_2205_13603_b200.runner import B200Runner  # noqa: E402

workload, family = sys.argv[1], sys.argv[2]
DT = sys.argv[3] if len(sys.argv) > 3 else ("f32" if workload.startswith("gmm512") else "bf16")
hdr, pop = load_population(workload)
progs = [p["program"] for p in pop]
probe = B200Runner(dtype=DT, min_repeats=50, max_repeats=2000, target_ms=0.5, timeout_ms=5.0)
probe.set_workload(hdr["e0"])
plans = probe.plan_programs(progs)
idx = [i for i, p in enumerate(plans) if p["family"] == family and p["status"] == "OK"]
res = probe.measure_programs([progs[i] for i in idx])
probe.close()
seen, top = set(), []
for j in sorted(range(len(idx)), key=lambda j: res[j]["latency_ns"] if res[j]["status"] == "OK" else 1e30):
    k = tuple(plans[idx[j]]["cfg"])
    if res[j]["status"] == "OK" and k not in seen:
        seen.add(k)
        top.append(idx[j])
    if len(top) == 4:
        break
print("cfg | us/launch at min_repeats 50, 200, 800, 2000")
rows = {i: [] for i in top}
for reps in (50, 200, 800, 2000):
    r = B200Runner(dtype=DT, min_repeats=reps, max_repeats=reps, target_ms=0.0, timeout_ms=5.0)
    r.set_workload(hdr["e0"])
    out = r.measure_programs([progs[i] for i in top])
    r.close()
    for i, x in zip(top, out):
        rows[i].append(x["latency_ns"] / 1e3 if x["status"] == "OK" else float("nan"))
for i in top:
    print(plans[i]["cfg"], " ".join(f"{v:6.3f}" for v in rows[i]))
