"""Per-configuration latency of one kernel family of a population, each
distinct configuration measured in its own measure call with >= 100
back-to-back timed repeats (the bench's best-schedule method):
  python scripts/family_best.py conv2d tcgen05_conv"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from conftest import load_population  # noqa: E402
from paper_2205_13603_b200.runner import B200Runner  # noqa: E402
import bench  # noqa: E402

workload, family = sys.argv[1], sys.argv[2]
hdr, pop = load_population(workload)
flops = bench.contraction_flops(hdr["e0"])
r = B200Runner(dtype="f32" if workload == "gmm512" else "bf16", min_repeats=100, max_repeats=2000, target_ms=0.5,
               timeout_ms=5.0)
r.set_workload(hdr["e0"])
progs = [p["program"] for p in pop]
plans = r.plan_programs(progs)
seen, rows = set(), []
for i, p in enumerate(plans):
    if p["family"] != family or p["status"] != "OK" or tuple(p["cfg"]) in seen:
        continue
    seen.add(tuple(p["cfg"]))
    x, = r.measure_programs([progs[i]])
    rows.append((x["latency_ns"] / 1e3, x["status"], x["repeats"], p["cfg"]))
for us, st, reps, cfg in sorted(rows):
    print(f"{us:8.2f} us {flops / us / 1e6:8.1f} TF/s  {st} reps {reps} cfg {cfg}")
