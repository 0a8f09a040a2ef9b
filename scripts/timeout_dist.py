import sys, os, statistics
sys.path.insert(0, "."); sys.path.insert(0, "tests")
from conftest import load_population
from paper_2205_13603_b200.runner import B200Runner
hdr, pop = load_population("bert_ffn")
r = B200Runner(dtype="bf16", min_repeats=3, max_repeats=200, target_ms=0.2, timeout_ms=0.9,
               timeout_factor=10.0, timeout_floor_ms=0.05, single_shot_factor=5.0)
r.set_workload(hdr["e0"])
texts = [p["program"] for p in pop[:1024]]
for rep in range(2):
    res = r.measure_programs(texts)
to = sorted(x["latency_ns"] / 1e3 for x in res if x["status"] == "TIMEOUT")
ok = sorted(x["latency_ns"] / 1e3 for x in res if x["status"] == "OK")
print("TIMEOUT n", len(to), "us quantiles", [round(to[int(q * (len(to) - 1))], 1) for q in (0, .1, .5, .9, 1)])
print("OK n", len(ok), "best", ok[:3], "device ms", r.elapsed_ms())
chk = sorted(x.get("checked_ns", 0) / 1e3 for x in res if x["status"] == "OK")
print("checked launch us (OK) lowest", [round(v, 1) for v in chk[:5]])
