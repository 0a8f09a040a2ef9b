"""conv2d population: per-family best latency (tcgen05 conv vs SIMT-A) and
parity of every tcgen05 conv candidate."""
import collections
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from conftest import load_population  # noqa: E402
from paper_2205_13603_b200.runner import B200Runner  # noqa: E402

hdr, pop = load_population("conv2d")
r = B200Runner(dtype="bf16", timeout_ms=50)
r.set_workload(hdr["e0"], seed=0)
progs = [p["program"] for p in pop]
res = r.measure_programs(progs)
print("statuses", collections.Counter((x["family"], x["status"]) for x in res))
best = {}
for i, x in enumerate(res):
    if x["status"] == "OK":
        f = x["family"]
        if f not in best or x["latency_ns"] < best[f][0]:
            best[f] = (x["latency_ns"], x["cfg"][:11], x["repeats"])
for f, v in sorted(best.items(), key=lambda kv: kv[1][0]):
    print(f"{f:14s} best {v[0] / 1e3:9.2f} us cfg {v[1]} reps {v[2]}")
tc = sorted((x["latency_ns"], x["cfg"][:7], x["mismatches"]) for x in res if x["family"] == "tcgen05_conv")
for t in tc:
    print("tcconv", round(t[0] / 1e3, 2), t[1], "mism", t[2])
