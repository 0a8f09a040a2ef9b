"""Run a few conv2d candidates of given families/cfg prefixes (for ncu launch lists)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
from conftest import load_population
from paper_2205_13603_b200.runner import B200Runner
hdr, pop = load_population("conv2d")
progs = [p["program"] for p in pop]
r = B200Runner(dtype="bf16", min_repeats=1, max_repeats=1, target_ms=0.001,
               timeout_ms=float(os.environ.get("TMO", "50")), timeout_factor=float(os.environ.get("TF", "0")))
r.set_workload(hdr["e0"], seed=0)
plans = r.plan_programs(progs)
sel = []
for spec in sys.argv[1:]:
    fam, *cfg = spec.split(":")
    want = [int(x) for x in cfg[0].split(",")] if cfg else []
    sel += [i for i, p in enumerate(plans) if p["family"] == fam and p["status"] == "OK"
            and p["cfg"][:len(want)] == want][:2]
res = r.measure_programs([progs[i] for i in sel])
for i, x in zip(sel, res):
    print(x["family"], x["status"], round(x["latency_ns"] / 1e3, 1), "us", x["cfg"][:8])
