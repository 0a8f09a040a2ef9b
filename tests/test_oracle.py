"""The CPU oracle against the reference's own golden outputs (parity pinning)."""
import json
import os
from fractions import Fraction

import numpy as np
import pytest

from conftest import GOLDEN, load_model, load_population, load_programs
from oracle import oracle as O


@pytest.fixture(scope="module")
def programs():
    return load_programs()


def test_latency_exact_on_goldens(programs):
    for r in programs:
        assert O.sim_latency(r["program"]) == Fraction(*r["latency"]), r["name"]


def test_hand_values(programs):
    # the reference's hand-computed cases (tests/test_machine.py:17-76)
    by = {r["name"]: r for r in programs}
    for name, want in [("hand_base_3", 3), ("hand_relu1024_3072", 3072),
                       ("hand_relu_sched_192", 192), ("hand_gmm4_400", 400),
                       ("hand_mma4_56", 56), ("hand_gmm16_24832", 24832),
                       ("hand_gmm64_5304768", 5304768), ("hand_copy_512", 512),
                       ("hand_copy_vec_64", 64)]:
        assert O.sim_latency(by[name]["program"]) == want


def test_features_bit_exact(programs):
    for r in programs:
        assert np.array_equal(O.featurize(r["program"]), np.array(r["features"])), r["name"]


def test_predict_matches_reference(programs):
    model = load_model()
    for r in programs:
        assert O.predict(r["features"], model) == pytest.approx(r["predicted"], rel=1e-12)
    # unfit model conventions (src/costmodel.py:98-100)
    assert O.predict([0.0] * 9, {"weights": None}) == 1.0
    assert O.predict([0.0] * 9, {"weights": None, "intercept": np.log(8.0),
                                 "n_records": 2}) == pytest.approx(8.0)


@pytest.mark.parametrize("name", ["bert_ffn", "bmm_qk", "gmm512", "conv2d"])
def test_population_batch(name):
    hdr, pop = load_population(name)
    num, den, feats, _, st = O.batch([p["program"] for p in pop], threads=4)
    assert (st == 0).all()
    for a, b, p in zip(num, den, pop):
        assert Fraction(int(a), int(b)) == Fraction(*p["latency"])
    assert np.array_equal(feats, np.array([p["features"] for p in pop]))


def test_output_oracle_matches_interpreter():
    z = np.load(os.path.join(GOLDEN, "outputs_small.npz"))
    for name in ("gmm", "bmm", "conv2d", "dense_relu"):
        e0 = bytes(z[f"{name}/e0"]).decode()
        for seed in (0, 1):
            ins = {k.split("/")[-1]: z[k] for k in z.files if k.startswith(f"{name}/s{seed}/in/")}
            outs = {k.split("/")[-1]: z[k] for k in z.files if k.startswith(f"{name}/s{seed}/out/")}
            got = O.reference_outputs(e0, ins)
            for k, v in outs.items():
                assert np.array_equal(got[k].astype(np.int64), v), (name, seed, k)


def test_output_oracle_pinned_at_baseline_shapes():
    """The numpy output oracle and the repo's random_inputs at the full
    BASELINE shapes (every config-5 task included) against sha256 hashes of
    the reference interpreter's own inputs and outputs
    (tests/golden/outputs_big.json, made by make_goldens.py outputs_big from
    `interp.random_inputs` / `interp.run`, `src/interp.py:54-63`, `:314-342`)."""
    import hashlib
    import json
    from paper_2205_13603_b200.inputs import random_inputs
    with open(os.path.join(GOLDEN, "outputs_big.json")) as fh:
        doc = json.load(fh)
    assert len(doc) == 7
    sha = lambda a: hashlib.sha256(np.ascontiguousarray(a, dtype=np.int64).tobytes()).hexdigest()
    for name, case in doc.items():
        ins = random_inputs(case["e0"], case["seed"])
        assert {k: sha(v) for k, v in ins.items()} == case["inputs"], name
        got = O.reference_outputs(case["e0"], ins)
        for k, want in case["outputs"].items():
            v = got[k]
            assert list(v.shape) == want["shape"], name
            assert np.array_equal(v, np.round(v)) and np.abs(v).max() == want["max_abs"], name
            assert sha(v) == want["sha256"], (name, k)
