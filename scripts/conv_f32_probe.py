"""fp32 conv2d: per-family best latency of the committed conv2d population in
fp32 (3xTF32 tcgen05_conv vs SIMT-A), every candidate timed with >= 100
chained launches (scripts/family_best.py method):
  python scripts/conv_f32_probe.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from conftest import load_population  # noqa: E402
from paper_2205_13603_b200.runner import B200Runner  # noqa: E402
import bench  # noqa: E402

hdr, pop = load_population("conv2d")
flops = bench.contraction_flops(hdr["e0"])
progs = [p["program"] for p in pop[:2048]]
r = B200Runner(dtype="f32", min_repeats=3, max_repeats=20, target_ms=0.05, timeout_ms=5.0)
r.set_workload(hdr["e0"])
res = r.measure_programs(progs)
r.close()
best = {}
for i, x in enumerate(res):
    if x["status"] == "OK":
        f = x["family"]
        best.setdefault(f, []).append((x["latency_ns"], i))
r = B200Runner(dtype="f32", min_repeats=100, max_repeats=2000, target_ms=0.5, timeout_ms=5.0)
r.set_workload(hdr["e0"])
for f, lst in sorted(best.items()):
    lst.sort()
    fin = r.measure_programs([progs[i] for _, i in lst[:6]])
    ok = [(x["latency_ns"], x["cfg"][:8]) for x in fin if x["status"] == "OK"]
    if ok:
        ns, cfg = min(ok)
        print(f"{f:14s} best {ns / 1e3:8.2f} us {flops / ns / 1e3:6.1f} TF/s cfg {cfg} ({len(lst)} OK in the slice)")
r.close()
