"""The tcgen05 tile on fp32 workloads (3xTF32, `csrc/tc_gemm.cu` X3): every
distinct configuration bit-exact against the oracle on the reference's integer
inputs after chained launches, and fp32-accurate on N(0,1) inputs (north_star:
fp32 rtol 1e-4), next to the SIMT family's own fp32 error."""
import numpy as np
import pytest

from conftest import load_population
from oracle import oracle as O
from paper_2205_13603_b200.inputs import normal_inputs, random_inputs

pytestmark = pytest.mark.gpu


def make_runner(**kw):
    from paper_2205_13603_b200.runner import B200Runner
    kw.setdefault("min_repeats", 1)
    kw.setdefault("max_repeats", 3)
    kw.setdefault("target_ms", 0.005)
    return B200Runner(device=0, dtype="f32", **kw)


@pytest.mark.parametrize("name", ["gmm512_tc", "bmm_qk", "bert_ffn"])
def test_every_3xtf32_configuration_exact_after_chained_launches(name):
    hdr, pop = load_population(name)
    e0 = hdr["e0"]
    progs = [p["program"] for p in pop]
    r = make_runner(min_repeats=8, max_repeats=8, timeout_ms=50.0)
    r.set_workload(e0, seed=2)
    want = next(iter(O.reference_outputs(e0, random_inputs(e0, 2)).values()))
    plans = r.plan_programs(progs)
    seen = {}
    for i, p in enumerate(plans):
        if p["family"] == "tcgen05" and p["status"] == "OK":
            assert p["cfg"][8] == 1, p
            seen.setdefault(tuple(p["cfg"]), i)
    assert len(seen) >= (20 if name == "gmm512_tc" else 4), len(seen)
    for cfg, i in seen.items():
        res, = r.measure_programs([progs[i]])
        assert res["status"] == "OK" and res["mismatches"] == 0 and res["repeats"] == 8, (cfg, res)
        assert np.array_equal(r.last_output().astype(np.float64), want), cfg
    r.close()


def test_3xtf32_fp32_accuracy_on_normal_inputs():
    hdr, pop = load_population("gmm512_tc")
    e0 = hdr["e0"]
    ins = normal_inputs(e0, 7)
    cast = {k: v.astype(np.float32) for k, v in ins.items()}
    want = next(iter(O.reference_outputs(e0, cast).values()))
    scale = np.abs(want).max()
    r = make_runner(rtol=1e-4, atol=1e-4 * scale, timeout_ms=50.0)
    r.set_workload(e0, inputs=ins)
    plans = r.plan_programs([p["program"] for p in pop[:2048]])
    err = {}
    for fam in ("tcgen05", "simt"):
        idx = [i for i, p in enumerate(plans) if p["family"] == fam and p["status"] == "OK"][:8]
        assert len(idx) == 8, fam
        e = []
        for i in idx:
            res, = r.measure_programs([pop[i]["program"]])
            assert res["status"] == "OK", (fam, res)
            out = r.last_output().astype(np.float64)
            np.testing.assert_allclose(out, want, rtol=1e-4, atol=1e-4 * scale)
            e.append(np.abs(out - want).max() / scale)
        err[fam] = max(e)
    # fp32-level error: a few ulps of the output scale, well inside the
    # north_star fp32 rtol 1e-4 (measured: 3xTF32 and fp32 FFMA both ~1e-6)
    print("max |err| / max |C|:", err)
    assert err["tcgen05"] < 1e-5, err
    assert err["tcgen05"] < 8 * err["simt"] + 1e-7, err
    r.close()


def test_3xtf32_conv_configurations_exact_and_fp32_accurate():
    # fp32 conv2d: every tcgen05_conv program (cfg[7] = 1: 3xTF32 halves of
    # the activation -- split once for a workload input, on every launch for
    # a pad stage's output -- and of the K-major weights) bit-exact after 8
    # chained launches on integer inputs, and within fp32 tolerance on N(0,1)
    hdr, pop = load_population("conv2d")
    e0 = hdr["e0"]
    progs = [p["program"] for p in pop]
    r = make_runner(min_repeats=8, max_repeats=8, timeout_ms=50.0)
    r.set_workload(e0, seed=2)
    want = next(iter(O.reference_outputs(e0, random_inputs(e0, 2)).values()))
    plans = r.plan_programs(progs)
    seen = {}
    for i, p in enumerate(plans):
        if p["family"] == "tcgen05_conv" and p["status"] == "OK":
            assert p["cfg"][7] == 1, p
            seen[(tuple(p["cfg"]), i)] = i
    assert len(seen) >= 20, len(seen)
    for cfg, i in seen.items():
        res, = r.measure_programs([progs[i]])
        assert res["status"] == "OK" and res["mismatches"] == 0 and res["repeats"] == 8, (cfg, res)
        assert np.array_equal(r.last_output().astype(np.float64), want), cfg
    r.close()
    ins = normal_inputs(e0, 7)
    want = next(iter(O.reference_outputs(e0, {k: v.astype(np.float32) for k, v in ins.items()}).values()))
    scale = np.abs(want).max()
    r = make_runner(rtol=1e-4, atol=1e-4 * scale, timeout_ms=50.0)
    r.set_workload(e0, inputs=ins)
    for cfg, i in list(seen.items())[:4]:
        res, = r.measure_programs([progs[i]])
        assert res["status"] == "OK", (cfg, res)
        out = r.last_output().astype(np.float64)
        np.testing.assert_allclose(out, want, rtol=1e-4, atol=1e-4 * scale)
        assert np.abs(out - want).max() / scale < 1e-5, cfg
    r.close()
