import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
from conftest import load_population
from oracle import oracle as O
from paper_2205_13603_b200.inputs import random_inputs
from paper_2205_13603_b200.runner import B200Runner
hdr, pop = load_population("conv2d")
e0 = hdr["e0"]
want = O.reference_outputs(e0, random_inputs(e0, 0))["O"]
progs = [p["program"] for p in pop]
for reps in (1, 2, 3):
    r = B200Runner(dtype="bf16", min_repeats=reps, max_repeats=reps, target_ms=0.001, timeout_ms=200)
    r.set_workload(e0, seed=0)
    plans = r.plan_programs(progs)
    i = next(i for i, p in enumerate(plans) if p["family"] == "simt_affine" and p["status"] == "OK")
    res, = r.measure_programs([progs[i]])
    out = r.last_output()
    print(reps, res["status"], res["mismatches"], res["repeats"], "nan", int(np.isnan(out).sum()), "eq", np.array_equal(out.astype(np.float64), want))
    r.close()
