"""Measure every tcgen05 candidate of a population with long graph repeats
(removes graph-launch overhead from the per-launch latency) and print them
sorted -- used to study the family's design space."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from conftest import load_population  # noqa: E402
from paper_2205_13603_b200.runner import B200Runner  # noqa: E402
import bench  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="bert_ffn")
ap.add_argument("--family", default="tcgen05")
ap.add_argument("--top", type=int, default=30)
ap.add_argument("--target-ms", type=float, default=0.5)
args = ap.parse_args()
hdr, pop = load_population(args.workload)
flops = bench.contraction_flops(hdr["e0"])
r = B200Runner(dtype="f32" if args.workload == "gmm512" else "bf16", min_repeats=20, max_repeats=400,
               target_ms=args.target_ms, timeout_ms=5)
r.set_workload(hdr["e0"])
progs = [p["program"] for p in pop]
plans = r.plan_programs(progs)
idx = [i for i, p in enumerate(plans) if p["family"].startswith(args.family) and p["status"] == "OK"]
seen, uniq = set(), []
for i in idx:
    k = tuple(plans[i]["cfg"])
    if k not in seen:
        seen.add(k)
        uniq.append(i)
res = r.measure_programs([progs[i] for i in uniq])
rows = sorted(zip(res, uniq), key=lambda x: x[0]["latency_ns"])
print(f"{len(idx)} {args.family} candidates, {len(uniq)} distinct cfgs")
for x, i in rows[:args.top]:
    us = x["latency_ns"] / 1e3
    print(f"{us:8.2f} us {flops / us / 1e6:8.1f} TF/s  {x['status']} reps {x['repeats']} cfg {plans[i]['cfg']}")
