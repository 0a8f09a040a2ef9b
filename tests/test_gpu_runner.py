"""The hardware Runner: every candidate's output against the oracle, per
kernel family, at the BASELINE shapes; float tolerance checks; statuses."""
import numpy as np
import pytest

from conftest import load_population
from oracle import oracle as O
from paper_2205_13603_b200.inputs import normal_inputs, random_inputs

pytestmark = pytest.mark.gpu


def make_runner(dtype, **kw):
    from paper_2205_13603_b200.runner import B200Runner
    kw.setdefault("min_repeats", 1)
    kw.setdefault("max_repeats", 3)
    kw.setdefault("target_ms", 0.005)
    return B200Runner(device=0, dtype=dtype, **kw)


def pick(plans, family, k):
    return [i for i, p in enumerate(plans) if p["family"] == family and p["status"] == "OK"][:k]


@pytest.mark.parametrize("name,dtype", [("bert_ffn", "bf16"), ("bmm_qk", "bf16"), ("gmm512", "f32"),
                                        ("bmm_qk", "f32")])
def test_reference_output_is_exact(name, dtype):
    hdr, _ = load_population(name)
    e0 = hdr["e0"]
    r = make_runner(dtype)
    r.set_workload(e0, seed=0)
    want = next(iter(O.reference_outputs(e0, random_inputs(e0, 0)).values()))
    assert np.array_equal(r.reference_output(), want)
    r.close()


@pytest.mark.parametrize("name,dtype,families", [
    ("bert_ffn", "bf16", ("tcgen05", "simt", "naive")),
    ("bmm_qk", "bf16", ("tcgen05", "simt")),
    ("gmm512", "f32", ("simt",)),
])
def test_candidates_bit_exact_per_family(name, dtype, families):
    hdr, pop = load_population(name)
    e0 = hdr["e0"]
    progs = [p["program"] for p in pop[:1024]] + [e0]
    r = make_runner(dtype, timeout_ms=50.0)
    r.set_workload(e0, seed=0)
    want = next(iter(O.reference_outputs(e0, random_inputs(e0, 0)).values()))
    plans = r.plan_programs(progs)
    for fam in families:
        idx = pick(plans, fam, 12 if fam != "naive" else 1)
        assert idx, fam
        for i in idx:
            res, = r.measure_programs([progs[i]])
            assert res["status"] == "OK", (fam, res)
            assert res["mismatches"] == 0 and res["max_abs_err"] == 0.0
            assert np.array_equal(r.last_output().astype(np.float64), want), (fam, res["cfg"])
    r.close()


def test_all_tcgen05_candidates_exact_bert_ffn():
    hdr, pop = load_population("bert_ffn")
    e0 = hdr["e0"]
    progs = [p["program"] for p in pop]
    r = make_runner("bf16")
    r.set_workload(e0, seed=1)
    plans = r.plan_programs(progs)
    idx = pick(plans, "tcgen05", 10 ** 6)
    res = r.measure_programs([progs[i] for i in idx])
    assert len(res) >= 60  # the whole tcgen05 space of this shape is ~100 programs
    for x in res:
        assert x["status"] == "OK" and x["mismatches"] == 0, x
        assert x["latency_ns"] > 0 and x["repeats"] >= 1
    r.close()


@pytest.mark.parametrize("name,family", [("bert_ffn", "tcgen05"), ("bmm_qk", "tcgen05"),
                                         ("conv2d", "tcgen05_conv")])
def test_tcgen05_back_to_back_repeats_exact(name, family):
    # C after a CUDA graph of 8 back-to-back launches (PDL chain, split-K
    # arrival tickets and in-kernel zeroing across launches) of every distinct
    # tcgen05 GEMM / conv configuration equals the oracle bit for bit
    hdr, pop = load_population(name)
    e0 = hdr["e0"]
    progs = [p["program"] for p in pop]
    r = make_runner("bf16", min_repeats=8, max_repeats=8)
    r.set_workload(e0, seed=2)
    want = next(iter(O.reference_outputs(e0, random_inputs(e0, 2)).values()))
    plans = r.plan_programs(progs)
    seen = {}
    for i, p in enumerate(plans):
        if p["family"] == family and p["status"] == "OK":
            seen.setdefault(tuple(p["cfg"]), i)
    assert seen
    for cfg, i in seen.items():
        res, = r.measure_programs([progs[i]])
        assert res["status"] == "OK" and res["mismatches"] == 0 and res["repeats"] == 8, (cfg, res)
        assert np.array_equal(r.last_output().astype(np.float64), want), cfg
    r.close()


def test_float_inputs_tolerance():
    # N(0,1) inputs: fp32 candidates within rtol 1e-4 of fp64 math; bf16 inputs
    # are rounded once at upload, the candidates then accumulate in fp32.
    for name, dtype, rtol in (("gmm512", "f32", 1e-4), ("bert_ffn", "bf16", 2e-2)):
        hdr, pop = load_population(name)
        e0 = hdr["e0"]
        ins = normal_inputs(e0, 7)
        r = make_runner(dtype, rtol=rtol, atol=1e-3, timeout_ms=50.0)
        r.set_workload(e0, inputs=ins)
        ref = r.reference_output()
        cast = {k: (v.astype(np.float32) if dtype == "f32" else
                    _bf16(v)) for k, v in ins.items()}
        want = next(iter(O.reference_outputs(e0, cast).values()))
        np.testing.assert_allclose(ref, want, rtol=1e-9, atol=1e-9)
        plans = r.plan_programs([p["program"] for p in pop[:600]])
        for fam in ("simt", "tcgen05"):
            for i in pick(plans, fam, 4):
                res, = r.measure_programs([pop[i]["program"]])
                assert res["status"] == "OK", res
                out = r.last_output().astype(np.float64)
                np.testing.assert_allclose(out, want, rtol=rtol, atol=1e-3)
        r.close()


def test_float_inputs_tolerance_conv2d_and_bmm():
    # the general path (pad stage + implicit GEMM) and batch matmul with N(0,1)
    # inputs: bf16 rtol 2e-2 (inputs rounded once at upload, fp32 accumulation)
    for name, fams in (("conv2d", ("tcgen05_conv", "simt_affine")), ("bmm_qk", ("tcgen05", "simt"))):
        hdr, pop = load_population(name)
        e0 = hdr["e0"]
        ins = normal_inputs(e0, 11)
        r = make_runner("bf16", rtol=2e-2, atol=1e-2, timeout_ms=1000.0)
        r.set_workload(e0, inputs=ins)
        want = next(iter(O.reference_outputs(e0, {k: _bf16(v) for k, v in ins.items()}).values()))
        np.testing.assert_allclose(r.reference_output(), want, rtol=1e-9, atol=1e-9)
        progs = [p["program"] for p in pop]
        plans = r.plan_programs(progs)
        for fam in fams:
            idx = pick(plans, fam, 3)
            assert len(idx) == 3, fam
            for i in idx:   # every pick must run to completion and pass
                res, = r.measure_programs([progs[i]])
                assert res["status"] == "OK", res
                np.testing.assert_allclose(r.last_output().astype(np.float64), want, rtol=2e-2, atol=1e-2)
        r.close()


def _bf16(v):
    import torch
    return torch.tensor(v, dtype=torch.float32).to(torch.bfloat16).to(torch.float32).numpy()


def test_statuses_and_sentinels():
    hdr, pop = load_population("bert_ffn")
    e0 = hdr["e0"]
    r = make_runner("bf16", timeout_ms=0.05)
    r.set_workload(e0, seed=0)
    progs = [p["program"] for p in pop[:400]]
    plans = r.plan_programs(progs)
    ill = [i for i, p in enumerate(plans) if p["status"] == "ILLEGAL"][:3]
    nest = [i for i, p in enumerate(plans) if p["family"] == "loopnest"][:1]
    res = r.measure_programs([progs[i] for i in ill + nest] + ["{bad"])
    assert [x["status"] for x in res[:len(ill)]] == ["ILLEGAL"] * len(ill)
    if nest:
        assert res[len(ill)]["status"] == "TIMEOUT"  # the PVU row-per-thread nest takes ms
    assert res[-1]["status"] == "PARSE"
    lats = r.latencies(res)
    base = r.baseline()
    sentinel = base * 10 ** 4  # finite, never inf (fit takes log latency)
    assert all(l == sentinel for l, x in zip(lats, res) if x["status"] != "TIMEOUT")
    for l, x in zip(lats, res):
        if x["status"] == "TIMEOUT":  # abort time: a lower bound above the deadline
            assert 0.05e6 <= float(l) <= float(sentinel)
    r.close()


def test_adaptive_timeout_bounds_slow_candidates():
    hdr, pop = load_population("bert_ffn")
    e0 = hdr["e0"]
    r = make_runner("bf16", timeout_ms=5.0, timeout_factor=10.0, timeout_floor_ms=0.02)
    r.set_workload(e0, seed=0)
    progs = [p["program"] for p in pop[:300]]
    plans = r.plan_programs(progs)
    fast = pick(plans, "tcgen05", 2)
    slow = pick(plans, "simt", 40)
    res = r.measure_programs([progs[i] for i in fast + slow])
    best = min(x["latency_ns"] for x in res if x["status"] == "OK")
    for x in res[len(fast):]:
        if x["status"] == "OK":
            assert x["mismatches"] == 0
        else:
            assert x["status"] == "TIMEOUT"
            # aborted near 10x the best checked run seen before it, far below the 5 ms cap
            assert x["latency_ns"] < 2.5e6
    assert any(x["status"] == "TIMEOUT" for x in res)
    r.close()


def test_measure_signature_matches_reference_runner():
    from fractions import Fraction
    hdr, pop = load_population("bmm_qk")
    r = make_runner("bf16")
    r.set_workload(hdr["e0"])

    class Cand:  # the reference Candidate's .program attribute (src/search.py:63-69)
        def __init__(self, p):
            self.program = p

    out = r.measure([Cand(p["program"]) for p in pop[:8]], None, 1)
    assert len(out) == 8 and all(isinstance(x, Fraction) and x > 0 for x in out)
    assert isinstance(r.baseline(), Fraction)
    r.close()


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_conv2d_general_path_bit_exact(dtype):
    """conv2d NHWC (pad stage + implicit GEMM): the fp64 reference run equals
    the numpy oracle; SIMT-A (pad stage separate and pad inlined as a guarded
    load), nest-generic, every tcgen05 conv candidate (TMA zero fill for the
    inlined pad, cluster split-K over filter rows) and the unscheduled e0
    match it bit-exactly."""
    import json
    hdr, pop = load_population("conv2d")
    e0 = hdr["e0"]
    r = make_runner(dtype, timeout_ms=2000.0)
    r.set_workload(e0, seed=0)
    want = O.reference_outputs(e0, random_inputs(e0, 0))["O"]
    assert np.array_equal(r.reference_output(), want)
    progs = [p["program"] for p in pop]
    plans = r.plan_programs(progs)
    inlined = [i for i, p in enumerate(progs)
               if len([b for b in json.loads(p)["buffers"]]) == 3 and plans[i]["status"] == "OK"
               and plans[i]["family"] != "nestgen"]
    # nest-generic candidates at this shape run the whole conv in <= 56
    # interpreted threads (seconds each); their bit-exactness is covered on the
    # ragged conv in test_gpu_e2e.py::test_ragged_shapes_every_candidate_exact
    picks = pick(plans, "simt_affine", 6) + inlined[:4]
    assert len(pick(plans, "simt_affine", 6)) == 6 and len(inlined) >= 4
    if dtype == "bf16":
        tc = [i for i, x in enumerate(plans) if x["family"] == "tcgen05_conv"]
        assert len(tc) >= 4
        picks += tc
    for i in picks:   # every pick must finish (2 s cap) and be bit-exact
        res, = r.measure_programs([progs[i]])
        assert res["status"] == "OK", res
        assert res["mismatches"] == 0, res
        assert np.array_equal(r.last_output().astype(np.float64), want), res["cfg"]
    base = r.baseline_result()
    assert base["status"] == "OK" and base["mismatches"] == 0
    r.close()


def test_conv2d_population_slice_has_no_parity_failures():
    # a bench-sized slice through every general-path family (AFFCOPY pad
    # stages incl. fused/vectorised pad loops, SIMT-A, NESTGEN, tcgen05 conv):
    # the in-run parity reducer flags no candidate
    hdr, pop = load_population("conv2d")
    e0 = hdr["e0"]
    r = make_runner("bf16", timeout_ms=20.0)
    r.set_workload(e0, seed=0)
    res = r.measure_programs([p["program"] for p in pop[:384]])
    bad = [x for x in res if x["status"] in ("PARITY", "LAUNCH")]
    assert not bad, bad[:3]
    assert sum(x["status"] == "OK" for x in res) > 50
    r.close()


def test_dense_relu_general_path_exact():
    from paper_2205_13603_b200.inputs import random_inputs as ri
    import gzip
    import json
    import os
    from conftest import GOLDEN
    rows = [json.loads(l) for l in open(os.path.join(GOLDEN, "programs.jsonl"))]
    progs = [x["program"] for x in rows if x["name"].startswith("dense_relu")]
    e0 = next(x["program"] for x in rows if x["name"] == "dense_relu_e0")
    r = make_runner("bf16", timeout_ms=200.0)
    r.set_workload(e0, seed=3)
    want = O.reference_outputs(e0, ri(e0, 3))["R"]
    assert np.array_equal(r.reference_output(), want)
    res = r.measure_programs(progs)
    ok = [x for x in res if x["status"] == "OK"]
    assert ok
    for x in res:
        if x["status"] == "OK":
            assert x["mismatches"] == 0, x
    r.close()


def test_sharded_runner_b200_workers_match_single_runner():
    # the real process-per-device path (two workers sharing GPU 0 here; one
    # per GPU on an 8-GPU box): dealt round-robin, gathered in candidate order
    from paper_2205_13603_b200.multigpu import ShardedRunner
    hdr, pop = load_population("bmm_qk")
    e0 = hdr["e0"]
    progs = [p["program"] for p in pop[:96]]
    one = make_runner("bf16", timeout_ms=5.0)
    one.set_workload(e0, seed=0)
    want = one.measure_programs(progs)
    one.close()
    sh = ShardedRunner([0, 0], dtype="bf16", min_repeats=1, max_repeats=3, target_ms=0.005,
                       timeout_ms=5.0)
    try:
        sh.set_workload(e0)
        got = sh.measure_programs(progs)
    finally:
        sh.close()
    assert len(got) == len(want)
    for g, w in zip(got, want):
        assert (g["family"], g["cfg"]) == (w["family"], w["cfg"])
        if w["status"] == "OK" and g["status"] == "OK":
            assert g["mismatches"] == 0
    assert sum(g["status"] == "OK" for g in got) >= 0.8 * sum(w["status"] == "OK" for w in want)


def test_single_shot_factor_skips_repeats_of_slow_candidates():
    hdr, pop = load_population("bmm_qk")
    e0 = hdr["e0"]
    progs = [p["program"] for p in pop[:128]]
    r = make_runner("bf16", timeout_ms=5.0, min_repeats=3, max_repeats=3, single_shot_factor=4.0)
    r.set_workload(e0, seed=0)
    res = r.measure_programs(progs)
    ok = [x for x in res if x["status"] == "OK"]
    best = min(x["latency_ns"] for x in ok)
    singles = [x for x in ok if x["repeats"] == 0]
    assert singles and all(x["mismatches"] == 0 for x in ok)
    assert all(x["latency_ns"] > 2.0 * best for x in singles)
    assert all(x["repeats"] == 3 for x in ok if x["latency_ns"] < 2.0 * best)
    r.close()


@pytest.mark.parametrize("name,dtype", [("bert_ffn", "bf16"), ("gmm512", "f32"), ("conv2d", "bf16"),
                                        ("conv2d", "f32")])
def test_set_workload_consumes_host_inputs_before_returning(name, dtype):
    """ls_runner_set_workload returns with the fp64 reference run still queued
    (include/loopsched_b200.h): the caller's host arrays must already be
    consumed, so overwriting them right after the call changes nothing --
    neither the reference output nor a candidate's parity verdict."""
    hdr, pop = load_population(name)
    e0 = hdr["e0"]
    ins = {k: np.ascontiguousarray(v, dtype=np.float32) for k, v in random_inputs(e0, 0).items()}
    outs = O.reference_outputs(e0, {k: v.copy() for k, v in ins.items()})
    want = outs["O"] if "O" in outs else next(iter(outs.values()))
    r = make_runner(dtype, timeout_ms=200.0)
    r.set_workload(e0, ins)
    for v in ins.values():
        v.fill(np.nan)   # the same buffers the C call read from
    plans = r.plan_programs([p["program"] for p in pop[:64]])
    ok = [i for i, p in enumerate(plans) if p["status"] == "OK"][:3]
    res = r.measure_programs([pop[i]["program"] for i in ok])
    assert np.array_equal(r.reference_output(), want)
    assert all(x["status"] in ("OK", "TIMEOUT") for x in res), res
    assert any(x["status"] == "OK" for x in res), res
    assert all(x["mismatches"] == 0 for x in res if x["status"] == "OK"), res
    r.close()


def test_simt_wide_register_tiles_and_chunked_k_tiles_exact():
    # round-2 instantiator coverage: register tiles 24/32/48/64 (the rest of
    # the 2^a 3^b lattice with RM x RN <= 64) and innermost K parts staged in
    # chunks when the whole part does not fit in shared memory -- both were
    # ILLEGAL by convention before; such candidates must be bit-exact
    hdr, pop = load_population("bert_ffn")
    e0 = hdr["e0"]
    progs = [p["program"] for p in pop[:1024]]
    r = make_runner("bf16", timeout_ms=200.0)
    r.set_workload(e0, seed=0)
    want = next(iter(O.reference_outputs(e0, random_inputs(e0, 0)).values()))
    plans = r.plan_programs(progs)
    simt = [i for i, p in enumerate(plans) if p["family"] == "simt" and p["status"] == "OK"]
    wide = [i for i in simt if max(plans[i]["cfg"][7], plans[i]["cfg"][8]) >= 24][:6]
    big = sorted(simt, key=lambda i: -plans[i]["cfg"][11])[:6]  # largest smem k-tiles (chunked ones among them)
    assert len(wide) == 6 and big
    ok = 0
    for i in dict.fromkeys(wide + big):
        res, = r.measure_programs([progs[i]])
        assert res["status"] in ("OK", "TIMEOUT"), res
        if res["status"] == "OK":
            ok += 1
            assert res["mismatches"] == 0
            assert np.array_equal(r.last_output().astype(np.float64), want), res["cfg"]
    assert ok >= 6
    r.close()


def test_traced_pipeline_depth_candidates_exact():
    # tcgen05 candidates of the pipelined b200 space (the unrolled inner
    # k-tile part = shared-memory stages in flight) are bit-exact for every
    # traced depth
    from paper_2205_13603_b200.refapi import loopsched
    from paper_2205_13603_b200.tensor_core import b200_space
    ls = loopsched()
    e0 = ls.ir.serialize(ls.gmm(128, 768, 3072))
    progs = [ls.ir.serialize(p) for p, _ in
             ls.spaces.sample_traces(ls.ir.deserialize(e0), b200_space(pipeline=True), 96, seed=11)]
    r = make_runner("bf16", timeout_ms=50.0)
    r.set_workload(e0, seed=0)
    want = next(iter(O.reference_outputs(e0, random_inputs(e0, 0)).values()))
    plans = r.plan_programs(progs)
    tc = [i for i, p in enumerate(plans) if p["family"] == "tcgen05" and p["status"] == "OK"]
    assert len({plans[i]["cfg"][6] for i in tc}) >= 3
    for i in tc:
        res, = r.measure_programs([progs[i]])
        assert res["status"] == "OK" and res["mismatches"] == 0, res
        assert np.array_equal(r.last_output().astype(np.float64), want), res["cfg"]
    r.close()


@pytest.mark.parametrize("name", ["bert_ffn", "bmm_qk"])
def test_cold_l2_timing_mode(name):
    # flush_l2: every timed repeat after a 256 MB scrub, timed alone; the
    # output after the repeats is still exact and a cold launch is no faster
    # than the same schedule's L2-warm chained launches
    hdr, pop = load_population(name)
    e0 = hdr["e0"]
    progs = [p["program"] for p in pop]
    warm = make_runner("bf16", min_repeats=50, max_repeats=50)
    warm.set_workload(e0, seed=3)
    plans = warm.plan_programs(progs)
    idx = pick(plans, "tcgen05", 3)
    assert idx
    w = warm.measure_programs([progs[i] for i in idx])
    warm.close()
    cold = make_runner("bf16", min_repeats=5, max_repeats=5, flush_l2=True)
    cold.set_workload(e0, seed=3)
    want = next(iter(O.reference_outputs(e0, random_inputs(e0, 3)).values()))
    for i, wx in zip(idx, w):
        cx, = cold.measure_programs([progs[i]])
        assert cx["status"] == "OK" and cx["mismatches"] == 0 and cx["repeats"] == 5, cx
        assert np.array_equal(cold.last_output().astype(np.float64), want)
        assert cx["latency_ns"] > 0.9 * wx["latency_ns"], (plans[i]["cfg"], cx["latency_ns"], wx["latency_ns"])
    cold.close()


def test_baseline_relative_deadline_cap():
    # baseline_timeout_factor: once e0 is measured, the checked-launch cap is
    # max(timeout_floor_ms, factor x baseline); with factor 0.1 a SIMT
    # candidate slower than that is aborted, and set_workload restores the
    # configured cap (the naive family has no deadline checks)
    hdr, pop = load_population("bert_ffn")
    e0 = hdr["e0"]
    progs = [p["program"] for p in pop]
    probe = make_runner("bf16", timeout_ms=50.0)
    probe.set_workload(e0, seed=0)
    plans = probe.plan_programs(progs)
    simt = pick(plans, "simt", 24)
    res = probe.measure_programs([progs[i] for i in simt])
    probe.close()
    slow = [i for i, x in zip(simt, res) if x["status"] == "OK" and x["latency_ns"] > 300e3]
    assert slow, "no SIMT candidate above 300 us in the slice"
    r = make_runner("bf16", timeout_ms=50.0, baseline_timeout_factor=0.1, timeout_floor_ms=0.05)
    r.set_workload(e0, seed=0)
    base_ns = float(r.baseline())
    cap_ns = max(50e3, 0.1 * base_ns)
    x, = r.measure_programs([progs[slow[0]]])
    assert x["status"] == "TIMEOUT", x
    assert x["latency_ns"] < 300e3 and x["latency_ns"] > 0.5 * cap_ns
    r.set_workload(e0, seed=0)
    y, = r.measure_programs([progs[slow[0]]])
    assert y["status"] == "OK" and y["mismatches"] == 0, y
    r.close()


def test_trace_tc_kernel_span():
    # per-CTA globaltimer stamps of one isolated tcgen05 launch: every CTA
    # stamped in order, the kernel's device span well under the events'
    # launch-to-launch time and the output still exact
    hdr, pop = load_population("bert_ffn")
    e0 = hdr["e0"]
    progs = [p["program"] for p in pop]
    r = make_runner("bf16")
    r.set_workload(e0, seed=0)
    plans = r.plan_programs(progs)
    i = next(i for i, p in enumerate(plans) if p["family"] == "tcgen05" and p["status"] == "OK"
             and p["cfg"][4] > 1)
    a = r.trace_tc(progs[i], 1)
    b, gm, gn, bn, splits = plans[i]["cfg"][:5]
    assert a.shape == (b * gm * gn * splits, 8)
    assert (a[:, 0] > 0).all() and (np.diff(a[:, [0, 1, 2, 3, 4, 6]], axis=1) >= 0).all()
    span = r.kernel_span_us(progs[i], samples=3)
    assert 0.5 < span < 200.0, span
    res, = r.measure_programs([progs[i]])
    assert res["status"] == "OK" and res["mismatches"] == 0
    r.close()


def test_launch_count_includes_set_workload_kernels():
    # the kernels set_workload enqueues (2 bf16 conversions, the fp64
    # reference, the K-major transpose) are reported once, by the next
    # measure call's launch count
    hdr, pop = load_population("bert_ffn")
    e0 = hdr["e0"]
    progs = [p["program"] for p in pop]
    r = make_runner("bf16", min_repeats=3, max_repeats=3)
    r.set_workload(e0, seed=0)
    i = next(i for i, p in enumerate(r.plan_programs(progs)) if p["family"] == "tcgen05" and p["status"] == "OK")
    r.measure_programs([progs[i]])
    first = r.launch_count()
    r.measure_programs([progs[i]])
    second = r.launch_count()
    assert first - second == 4, (first, second)
    r.close()
