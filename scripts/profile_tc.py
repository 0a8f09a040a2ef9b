"""Run selected candidates of a population through the runner (for ncu)."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from conftest import load_population  # noqa: E402
from paper_2205_13603_b200.runner import B200Runner  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="bert_ffn")
ap.add_argument("--family", default="tcgen05")
ap.add_argument("--count", type=int, default=8)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--cfg", default="")
ap.add_argument("--dtype", default="")
ap.add_argument("--host-us", type=float, default=0.0)  # comma list of cfg prefixes to select, e.g. "1,1,12,64,12"
args = ap.parse_args()
hdr, pop = load_population(args.workload)
dtype = args.dtype or ("f32" if args.workload.startswith("gmm512") else "bf16")
r = B200Runner(dtype=dtype, min_repeats=args.reps, max_repeats=args.reps, target_ms=0.001, timeout_ms=5)
r.set_workload(hdr["e0"])
progs = [p["program"] for p in pop]
plans = r.plan_programs(progs)
want = [int(x) for x in args.cfg.split(",")] if args.cfg else None
idx = [i for i, p in enumerate(plans) if p["family"] == args.family and p["status"] == "OK"
       and (want is None or p["cfg"][:len(want)] == want)][:args.count]
r.debug_stats(args.host_us)
res = r.measure_programs([progs[i] for i in idx])
print("stats", r.debug_stats(), "launches", r.launch_count(), "device ms", r.elapsed_ms())
for x in sorted(res, key=lambda x: x["latency_ns"]):
    print(x["family"], x["status"], f"{x['latency_ns']/1e3:.2f}us", x["cfg"][:8], "reps", x["repeats"])
