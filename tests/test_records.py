"""Hardware-latency record / report format (records.py),
driven through the reference's unchanged search on CPU with a runner that
returns nanosecond Fractions (the GPU runner's unit)."""
import hashlib
import json
from fractions import Fraction

import numpy as np
import pytest

from conftest import needs_reference

pytestmark = needs_reference


class NsRunner:
    """Runner protocol: a deterministic ns latency per program (the reference
    simulation scaled to a non-integer ns value) plus per-candidate results
    the way B200Runner.last_results reports them."""

    def __init__(self):
        from paper_2205_13603_b200.refapi import loopsched
        self.ls = loopsched()
        self.last_results = []

    def _ns(self, prog):
        return Fraction(self.ls.machine.simulate_latency(prog, self.ls.MachineSpec())) / 7 + Fraction(1, 1000)

    def measure(self, candidates, spec=None, jobs=1):
        out = [self._ns(c.program) for c in candidates]
        self.last_results = [{"family": "tcgen05", "cfg": [i, 1, 2], "status": "OK", "repeats": 3}
                             for i, _ in enumerate(candidates)]
        return out

    def baseline(self, e0, spec=None):
        return self._ns(e0)


class RefScorer:
    def __init__(self):
        from paper_2205_13603_b200.refapi import loopsched
        self.ls = loopsched()

    def featurize_batch(self, programs, spec=None):
        ir = self.ls.ir
        return np.stack([self.ls.costmodel.featurize(ir.deserialize(p), spec or self.ls.MachineSpec())
                         for p in programs])

    def score_batch(self, feats, model):
        return np.array([model.predict_features(f) for f in np.asarray(feats)])


def digest(report):
    return hashlib.sha256(json.dumps(report.to_json(timestamp=False), sort_keys=True).encode()).hexdigest()


def run(tmp_path, warm_path=None, out="rec.jsonl", seed=3):
    from paper_2205_13603_b200 import plugin
    from paper_2205_13603_b200.refapi import loopsched
    ls = loopsched()
    e0 = ls.gmm(64, 64, 64)
    cfg = ls.SearchConfig(trials=24, batch=8, population=16, seed=seed)
    return plugin.tune_with_records(e0, ls.default_space(), cfg, runner=NsRunner(), scorer=RefScorer(),
                                    records_path=str(tmp_path / out), warm_path=warm_path,
                                    peak_tflops=1668.5, peak_source="test")


def test_report_has_hardware_section(tmp_path):
    from paper_2205_13603_b200.records import contraction_flops
    from paper_2205_13603_b200.refapi import loopsched
    report, doc = run(tmp_path)
    hw = doc["hardware"]
    flops = contraction_flops(loopsched().gmm(64, 64, 64))
    assert flops == 2 * 64 ** 3 and hw["context"]["unit"] == "ns"
    best = report.best.latency
    assert hw["best"]["tflops"] == pytest.approx(flops / (float(best) * 1e-9) / 1e12, rel=1e-12)
    assert hw["best"]["roofline"]["frac"] == pytest.approx(hw["best"]["tflops"] / 1668.5)
    assert hw["best"]["family"] == "tcgen05" and len(hw["records"]) == len(report.log)
    # the reference's own keys are untouched
    assert {k for k in doc if k != "hardware"} == set(report.to_json(timestamp=False))


def test_records_round_trip_exact_and_warm_start(tmp_path):
    from paper_2205_13603_b200 import records as R
    from paper_2205_13603_b200.refapi import loopsched
    ls = loopsched()
    report, _ = run(tmp_path)
    ctx = R.HardwareContext.for_workload(ls.gmm(64, 64, 64))
    got = R.load_records(str(tmp_path / "rec.jsonl"), workload_hash=ctx.workload_hash, unit="ns")
    assert [g.latency for g in got] == [r.latency for r in report.log]        # exact Fractions
    assert all(g.latency.denominator > 1 for g in got)                      # sub-ns precision kept
    assert [g.program_hash for g in got] == [r.program_hash for r in report.log]
    assert all(np.array_equal(g.features, r.features) for g, r in zip(got, report.log))
    # warm start from the file == warm start from the in-memory log
    from paper_2205_13603_b200 import plugin
    e0 = ls.gmm(64, 64, 64)
    cfg = ls.SearchConfig(trials=16, batch=8, population=16, seed=9)
    a, _ = plugin.tune_with_records(e0, ls.default_space(), cfg, runner=NsRunner(), scorer=RefScorer(),
                                    warm_path=str(tmp_path / "rec.jsonl"))
    b = plugin.tune(e0, ls.default_space(), cfg, None, report.log, runner=NsRunner(), scorer=RefScorer())
    assert digest(a) == digest(b)


def test_records_refuse_other_unit_or_workload(tmp_path):
    from paper_2205_13603_b200 import records as R
    run(tmp_path)
    with pytest.raises(ValueError, match="unit"):
        R.load_records(str(tmp_path / "rec.jsonl"), unit="cycles")
    with pytest.raises(ValueError, match="workload"):
        R.load_records(str(tmp_path / "rec.jsonl"), workload_hash=12345)


def test_reference_record_files_still_load(tmp_path):
    # files written by the reference's own save_records (float latency, no unit)
    from paper_2205_13603_b200 import records as R
    from paper_2205_13603_b200.refapi import loopsched
    ls = loopsched()
    e0 = ls.gmm(32, 32, 32)
    rep = ls.tune(e0, ls.default_space(), ls.SearchConfig(trials=8, batch=4, population=8, seed=1))
    ls.search.save_records(str(tmp_path / "ref.jsonl"), rep.log)
    got = R.load_records(str(tmp_path / "ref.jsonl"), unit="cycles")
    assert [g.latency for g in got] == [r.latency for r in rep.log]


def test_roofline_bound_follows_the_best_family(tmp_path):
    # tcgen05 best -> tensor bound; an fp32 SIMT best -> fp32-simt bound
    _, doc = run(tmp_path)
    assert doc["hardware"]["best"]["roofline"]["bound"] == "tensor"
    from paper_2205_13603_b200.records import HardwareContext, report_json
    report, _ = run(tmp_path, out="rec2.jsonl")
    from paper_2205_13603_b200.refapi import loopsched
    ctx = HardwareContext.for_workload(loopsched().gmm(64, 64, 64), dtype="f32", peak_tflops=74.4,
                                       peak_source="fp32 SIMT nominal")
    simt = report_json(report, ctx, info={report.best.program_hash: {"family": "simt"}})
    assert simt["hardware"]["best"]["roofline"]["bound"] == "fp32-simt"
    x3 = report_json(report, ctx, info={report.best.program_hash: {"family": "tcgen05"}})
    assert x3["hardware"]["best"]["roofline"]["bound"] == "tensor"
