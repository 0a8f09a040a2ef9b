"""Parity at the config-5 (BERT-base end-to-end) task shapes that are not
bench workloads: dense gmm(128,768,768), FFN-in gmm(128,3072,768) and the
attention PV batch_matmul(12,128,64,128).  For each: the GPU's fp64
reference run of the unscheduled program equals the numpy oracle (itself
pinned to the reference interpreter by sha256, tests/golden/outputs_big.json,
tests/test_oracle.py), every tcgen05 schedule of the population and at least
12 SIMT schedules are bit-exact."""
import numpy as np
import pytest

from conftest import load_population
from oracle import oracle as O
from paper_2205_13603_b200.inputs import random_inputs

pytestmark = pytest.mark.gpu

CASES = ["bert_dense", "bert_ffn_in", "bmm_pv"]


def make_runner(**kw):
    from paper_2205_13603_b200.runner import B200Runner
    kw.setdefault("min_repeats", 1)
    kw.setdefault("max_repeats", 3)
    kw.setdefault("target_ms", 0.005)
    return B200Runner(device=0, dtype="bf16", **kw)


@pytest.mark.parametrize("name", CASES)
def test_config5_reference_output_equals_oracle(name):
    hdr, _ = load_population(name)
    e0 = hdr["e0"]
    r = make_runner()
    r.set_workload(e0, seed=0)
    want = next(iter(O.reference_outputs(e0, random_inputs(e0, 0)).values()))
    assert np.array_equal(r.reference_output(), want)
    base = r.baseline_result()
    assert base["status"] == "OK" and base["mismatches"] == 0
    r.close()


@pytest.mark.parametrize("name", CASES)
def test_config5_every_tcgen05_schedule_exact(name):
    hdr, pop = load_population(name)
    e0 = hdr["e0"]
    progs = [p["program"] for p in pop]
    r = make_runner(timeout_ms=50.0)
    r.set_workload(e0, seed=0)
    want = next(iter(O.reference_outputs(e0, random_inputs(e0, 0)).values()))
    plans = r.plan_programs(progs)
    idx = [i for i, p in enumerate(plans) if p["family"] == "tcgen05" and p["status"] == "OK"]
    assert idx, "no tcgen05 schedule in the population"
    res = r.measure_programs([progs[i] for i in idx])
    for x in res:   # in-run parity reducer against the fp64 reference == oracle
        assert x["status"] == "OK" and x["mismatches"] == 0 and x["max_abs_err"] == 0.0, x
    seen = set()
    for i in idx:   # one output per distinct configuration, compared on the host
        key = tuple(plans[i]["cfg"])
        if key in seen or len(seen) >= 6:
            continue
        seen.add(key)
        x, = r.measure_programs([progs[i]])
        assert x["status"] == "OK"
        assert np.array_equal(r.last_output().astype(np.float64), want), key
    r.close()


@pytest.mark.parametrize("name", CASES)
def test_config5_simt_schedules_exact(name):
    hdr, pop = load_population(name)
    e0 = hdr["e0"]
    progs = [p["program"] for p in pop]
    r = make_runner(timeout_ms=500.0)
    r.set_workload(e0, seed=0)
    want = next(iter(O.reference_outputs(e0, random_inputs(e0, 0)).values()))
    plans = r.plan_programs(progs)
    idx = [i for i, p in enumerate(plans) if p["family"] == "simt" and p["status"] == "OK"][:12]
    assert len(idx) == 12
    for i in idx:
        x, = r.measure_programs([progs[i]])
        assert x["status"] == "OK" and x["mismatches"] == 0, x
        assert np.array_equal(r.last_output().astype(np.float64), want), plans[i]["cfg"]
    r.close()
