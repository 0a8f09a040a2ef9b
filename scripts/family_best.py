"""Per-configuration latency of one kernel family of a population: every
candidate of the family measured in its own measure call with >= 100
back-to-back timed repeats (the bench's best-schedule method), the fastest
candidate per kernel configuration reported (a candidate's latency covers all
of its kernels, e.g. a separate pad stage before a conv):
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
best = {}
idx = [i for i, p in enumerate(plans) if p["family"] == family and p["status"] == "OK"]
batch = "--batch" in sys.argv  # all candidates in one measure call (as the bench's final re-measure)
res = r.measure_programs([progs[i] for i in idx]) if batch else [r.measure_programs([progs[i]])[0] for i in idx]
for i, x in zip(idx, res):
    p = plans[i]
    k = tuple(p["cfg"])
    if x["status"] == "OK" and (k not in best or x["latency_ns"] < best[k][0]):
        best[k] = (x["latency_ns"], x["repeats"], i)
for k, (ns, reps, i) in sorted(best.items(), key=lambda kv: kv[1][0]):
    us = ns / 1e3
    print(f"{us:8.2f} us {flops / us / 1e6:8.1f} TF/s  reps {reps} cfg {list(k)} program #{i}")
