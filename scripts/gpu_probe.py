"""Quick GPU probe used during development: cost kernels vs goldens, runner on
a slice of each population.  Prints a compact report."""
import json
import os
import sys
import time
from collections import Counter
from fractions import Fraction

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from conftest import load_model, load_population, load_programs  # noqa: E402
from paper_2205_13603_b200.runner import B200Runner  # noqa: E402
from paper_2205_13603_b200.scorer import GpuScorer  # noqa: E402

which = sys.argv[1:] or ["cost", "runner"]

if "cost" in which:
    rows = load_programs()
    model = load_model()
    sc = GpuScorer()
    t = time.time()
    lats, feats, pred = sc.analyze([r["program"] for r in rows], model=model)
    print("analyze", len(rows), f"{time.time()-t:.3f}s")
    bad_lat = [r["name"] for r, l in zip(rows, lats) if l != Fraction(*r["latency"])]
    F = np.array([r["features"] for r in rows])
    exact = (feats == F).all(axis=1)
    rel = np.abs(feats - F) / np.maximum(np.abs(F), 1e-300)
    print("latency mismatches", len(bad_lat), bad_lat[:5])
    print("features exact rows", int(exact.sum()), "/", len(rows), "max rel", float(rel.max()))
    P = np.array([r["predicted"] for r in rows])
    print("pred max rel", float(np.max(np.abs(pred - P) / P)))
    for name in ["bert_ffn", "bmm_qk", "gmm512", "conv2d"]:
        hdr, pop = load_population(name)
        lats, feats, _ = sc.analyze([p["program"] for p in pop])
        okl = all(l == Fraction(*p["latency"]) for l, p in zip(lats, pop))
        okf = np.array_equal(feats, np.array([p["features"] for p in pop]))
        print(name, "lat exact", okl, "feat exact", okf)

if "runner" in which:
    for name, dtype, take in [("bert_ffn", "bf16", 400), ("bmm_qk", "bf16", 200), ("gmm512", "f32", 200)]:
        hdr, pop = load_population(name)
        r = B200Runner(dtype=dtype, timeout_ms=2.0)
        t = time.time()
        r.set_workload(hdr["e0"])
        base = r.baseline_result()
        print(name, "baseline", base["status"], base["family"], f"{base['latency_ns']/1e3:.1f}us",
              "err", base["max_abs_err"], f"setup {time.time()-t:.2f}s")
        progs = [p["program"] for p in pop[:take]]
        t = time.time()
        res = r.measure_programs(progs)
        wall = time.time() - t
        c = Counter((x["family"], x["status"]) for x in res)
        print("  ", dict(c), f"wall {wall:.2f}s device {r.elapsed_ms():.1f}ms launches {r.launch_count()}")
        ok = [x for x in res if x["status"] == "OK"]
        best = sorted(ok, key=lambda x: x["latency_ns"])[:5]
        for b in best:
            print("   best", b["family"], f"{b['latency_ns']/1e3:.2f}us", b["cfg"], "reps", b["repeats"])
        par = [x for x in res if x["status"] == "PARITY"]
        for x in par[:5]:
            print("   PARITY", x["family"], x["cfg"], x["max_abs_err"], x["mismatches"])
        r.close()
