"""Native trace replay / validation (csrc/replay.cpp).

Parity against the reference's ``validate_trace`` (`src/trace.py:258-265`):
every committed replay vector (sampled and mutated traces of the four
population spaces, incl. rejections) must give the same verdict, the same
``ir.serialize`` program text, ``ir.structural_hash`` and normalized
``serialize_trace`` text, or the same (reason, index); and the reference's own
``tune`` with only the validator swapped for the native one must produce a
byte-identical report.  Host-only: no GPU needed."""
import gzip
import json
import os

import pytest

from conftest import GOLDEN, needs_reference

TASKS = ["bert_ffn", "bmm_qk", "gmm512", "conv2d"]


def load_replay(name):
    with gzip.open(os.path.join(GOLDEN, f"replay_{name}.jsonl.gz"), "rt") as fh:
        lines = fh.read().splitlines()
    return json.loads(lines[0]), [json.loads(l) for l in lines[1:]]


@pytest.mark.parametrize("name", TASKS)
def test_native_replay_matches_reference_vectors(name):
    from paper_2205_13603_b200.replay import ACCEPTED, REJECTED, NativeReplayer
    hdr, rows = load_replay(name)
    rp = NativeReplayer(hdr["e0"])
    out = rp.validate([r["trace"] for r in rows])
    assert len(out) == len(rows)
    for r, (st, idx, h, prog, norm, reason) in zip(rows, out):
        if r["accepted"]:
            assert st == ACCEPTED, (reason, r["trace"][:200])
            assert prog == r["program"]
            assert h == r["hash"]
            if "normalized" in r:
                assert norm == r["normalized"]
        else:
            assert st == REJECTED
            assert (reason, idx) == (r["reason"], r["index"])


def test_native_replay_single_and_batched_agree():
    from paper_2205_13603_b200.replay import NativeReplayer
    hdr, rows = load_replay("conv2d")
    rp = NativeReplayer(hdr["e0"])
    keys = [r["trace"] for r in rows[:40]]
    batch = rp.validate(keys)          # >= 32: host thread pool
    single = [rp.validate([k])[0] for k in keys]
    assert batch == single


def test_workload_hash_mismatch_is_rejected_at_minus_one():
    from paper_2205_13603_b200.replay import REJECTED, NativeReplayer
    hdr, rows = load_replay("gmm512")
    rp = NativeReplayer(hdr["e0"])
    t = '{"workload_hash": 12345}\n' + rows[0]["trace"]
    (st, idx, _h, _p, _n, reason), = rp.validate([t])
    assert (st, idx) == (REJECTED, -1)
    assert "structural hash mismatch" in reason


@needs_reference
def test_program_hash_and_lazy_program_match_reference():
    from paper_2205_13603_b200.refapi import loopsched
    from paper_2205_13603_b200.replay import lazy_program_class, program_hash
    ls = loopsched()
    hdr, rows = load_replay("bmm_qk")
    Lazy = lazy_program_class()
    for r in rows[:20]:
        p = ls.ir.deserialize(r["program"])
        assert program_hash(r["program"]) == ls.ir.structural_hash(p) == r["hash"]
        lp = Lazy(r["program"])
        assert isinstance(lp, ls.ir.TensorProgram)
        assert ls.ir.serialize(lp) == r["program"]
        assert ls.ir.structural_hash(lp) == r["hash"]
        assert lp == p


@needs_reference
@pytest.mark.parametrize("task", ["gmm512_default", "bert_ffn_b200"])
def test_tune_with_native_validator_is_byte_identical(task):
    # the reference's tune (simulated measurement, host featurize) with only
    # _Validator swapped: same trials, latencies, chosen trace, report
    from paper_2205_13603_b200 import plugin
    from paper_2205_13603_b200.refapi import loopsched
    from paper_2205_13603_b200.tensor_core import b200_space
    ls = loopsched()
    S = ls.search
    if task == "gmm512_default":
        e0 = ls.gmm(512, 512, 512)
        gen = ls.spaces.space_from_config({"modules": [{"mlt": {"structure": "SSRSR"}}, {"auto_inline": {}},
                                                       {"pvu": {"widths": [4, 8]}}]})
    else:
        e0, gen = ls.gmm(128, 768, 3072), b200_space()
    cfg = S.SearchConfig(trials=48, seed=0)
    ref = S.tune(e0, gen, cfg)
    with plugin.installed(native_replay=True, lookahead=False):
        assert S._Validator is not None and getattr(S._Validator, "_ls_dispatch", False)
        nat = S.tune(e0, gen, cfg)
    assert not getattr(S._Validator, "_ls_dispatch", False)  # restored
    a = json.dumps(ref.to_json(timestamp=False), sort_keys=True)
    b = json.dumps(nat.to_json(timestamp=False), sort_keys=True)
    assert a == b


@needs_reference
def test_lookahead_prefetch_keeps_the_tune_byte_identical():
    # the look-ahead replays every single-decision neighbour of each new
    # member and featurizes their programs ahead (here on the host: no GPU
    # scorer installed); the search must not change at all
    from paper_2205_13603_b200 import plugin
    from paper_2205_13603_b200.refapi import loopsched
    ls = loopsched()
    S = ls.search
    e0 = ls.gmm(64, 64, 64)
    gen = ls.spaces.space_from_config({"modules": [{"mlt": {"structure": "SSRSR"}}, {"auto_inline": {}},
                                                   {"pvu": {"widths": [4, 8]}}]})
    cfg = S.SearchConfig(trials=24, batch=8, population=12, generations=2, seed=3)
    ref = S.tune(e0, gen, cfg)
    with plugin.installed(native_replay=True, lookahead=True):
        nat = S.tune(e0, gen, cfg)
        v = plugin._current().validator
        assert v is not None and v.expansions > 0 and v.neighbours > 0 and v.prefetched > 0
    a = json.dumps(ref.to_json(timestamp=False), sort_keys=True)
    b = json.dumps(nat.to_json(timestamp=False), sort_keys=True)
    assert a == b


@needs_reference
@pytest.mark.parametrize("name", ["bert_ffn", "conv2d", "gmm512"])
def test_native_resample_equals_reference_resample(name):
    # replay(e0, t, mode="resample", seed): the native samplers draw from a
    # bit-exact port of CPython's random.Random(seed), so program, hash and
    # re-recorded trace equal the reference's for every seed
    from paper_2205_13603_b200.refapi import loopsched
    from paper_2205_13603_b200.replay import ACCEPTED, REJECTED, NativeReplayer
    ls = loopsched()
    hdr, rows = load_replay(name)
    e0 = ls.ir.deserialize(hdr["e0"])
    rp = NativeReplayer(hdr["e0"])
    n = 0
    for k, r in enumerate(rows[:24]):
        t = ls.trace.deserialize_trace(r["trace"])
        key = ls.trace.serialize_trace(t)
        for seed in (0, 1, 12345, 2 ** 40 + k, 2 ** 62 - 1 - k):
            st, idx, h, prog, norm, reason = rp.resample(key, seed)
            try:
                p, nt = ls.trace.replay(e0, t, mode="resample", seed=seed)
            except ls.trace.ReplayError as exc:
                assert st == REJECTED and (reason, idx) == (exc.reason, exc.index)
                continue
            assert st == ACCEPTED
            assert prog == ls.ir.serialize(p) and h == ls.ir.structural_hash(p)
            assert norm == ls.trace.serialize_trace(nt)
            n += 1
    assert n >= 60


@needs_reference
def test_lazy_program_pickles_by_text():
    import pickle
    from paper_2205_13603_b200.refapi import loopsched
    from paper_2205_13603_b200.replay import lazy_program_class
    ls = loopsched()
    text = ls.ir.serialize(ls.gmm(8, 8, 8))
    p = lazy_program_class()(text)
    q = pickle.loads(pickle.dumps(p))
    assert q == p and q._ls_text == text and ls.ir.serialize(q) == text


@needs_reference
@pytest.mark.parametrize("name", TASKS)
def test_cached_trace_serialization_equals_reference(name):
    # replay.serialize_trace caches each instruction's JSON line on the
    # instruction object; a chain of mutations (which share all but one
    # instruction with their parent) and normalized traces rebuilt from the
    # native text serialize byte-identically to the reference's
    import random
    from paper_2205_13603_b200.refapi import loopsched
    from paper_2205_13603_b200.replay import ACCEPTED, NativeReplayer, normalized_trace, serialize_trace
    ls = loopsched()
    hdr, rows = load_replay(name)
    rp = NativeReplayer(hdr["e0"])
    rng = random.Random(7)
    n = 0
    for r in rows[:16]:
        t = ls.trace.deserialize_trace(r["trace"])
        for _ in range(12):
            assert serialize_trace(t) == ls.trace.serialize_trace(t)
            key = serialize_trace(t)
            (st, _i, _h, _p, norm, _r), = rp.validate([key])
            if st == ACCEPTED:
                nt = normalized_trace(key, norm, t)
                assert serialize_trace(nt) == ls.trace.serialize_trace(nt) == norm
                n += 1
            t, _pos = ls.trace.mutate(t, rng)
    assert n >= 16
