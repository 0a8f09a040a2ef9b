"""Seam installation into the reference's unchanged search (CPU: the seams are
driven with the reference's own functions, so the tuning report must be
byte-identical; the GPU versions of runner/scorer are covered by -m gpu)."""
import hashlib
import json

import numpy as np
import pytest

from conftest import needs_reference

pytestmark = needs_reference


class RefRunner:
    """Runner protocol backed by the reference simulator."""

    def __init__(self):
        from paper_2205_13603_b200.refapi import loopsched
        self.ls = loopsched()
        self.calls = 0

    def measure(self, candidates, spec=None, jobs=1):
        self.calls += 1
        return [self.ls.machine.simulate_latency(c.program, spec) for c in candidates]

    def baseline(self, e0, spec=None):
        return self.ls.machine.simulate_latency(e0, spec)


class RefScorer:
    """Scorer protocol backed by the reference cost model."""

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


def test_installed_seams_preserve_every_decision():
    from paper_2205_13603_b200.refapi import loopsched
    from paper_2205_13603_b200 import plugin
    ls = loopsched()
    e0 = ls.gmm(64, 64, 64)
    cfg = ls.SearchConfig(trials=48, batch=8, population=16, seed=4)
    want = digest(ls.tune(e0, ls.default_space(), cfg))
    runner, scorer = RefRunner(), RefScorer()
    with plugin.installed(runner, scorer) as cache:
        got = digest(ls.tune(e0, ls.default_space(), cfg))
        assert cache.launches > 0
    assert got == want
    assert runner.calls > 0


def test_seams_restored_after_failure():
    from paper_2205_13603_b200.refapi import loopsched
    from paper_2205_13603_b200 import plugin
    ls = loopsched()
    before = (ls.search._measure_batch, ls.search.simulate_latency, ls.search.featurize,
              ls.search._Validator._predict)

    class Boom(RefRunner):
        def measure(self, *a, **k):
            raise RuntimeError("boom")

    with pytest.raises(RuntimeError):
        with plugin.installed(Boom(), RefScorer()):
            ls.search.tune(ls.gmm(8, 8, 8), ls.default_space(), ls.SearchConfig(trials=4, batch=2, population=4))
    after = (ls.search._measure_batch, ls.search.simulate_latency, ls.search.featurize,
             ls.search._Validator._predict)
    assert before == after


def test_golden_tune_reports_match_the_reference():
    # the committed tune goldens are the reference's own reports (make_goldens.py)
    import os
    from conftest import GOLDEN
    from paper_2205_13603_b200.refapi import loopsched
    ls = loopsched()
    doc = json.load(open(os.path.join(GOLDEN, "tune_gmm512.json")))
    assert doc["sha256"].startswith("45bd0d9a9c2f3be3")  # SURVEY.md §8c survey-time golden
    report = ls.tune(ls.gmm(512, 512, 512), ls.default_space(), ls.SearchConfig(trials=64, seed=0))
    assert digest(report) == doc["sha256"]


def test_positive_score_only_clamps_unusable_predictions():
    from paper_2205_13603_b200.plugin import positive_score
    assert positive_score(1.5) == 1.5 and positive_score(1e-300) == 1e-300
    assert positive_score(0.0) > 0.0 and positive_score(-0.0) > 0.0
    assert positive_score(float("inf")) < float("inf")
    assert positive_score(float("nan")) == positive_score(float("inf"))
