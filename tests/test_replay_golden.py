"""Trace-replay parity vectors (SURVEY.md §8f-1 groundwork).

``tests/golden/replay_<task>.jsonl.gz`` holds, per BASELINE population space,
sampled traces and single-decision mutations of them with the reference's
``validate_trace`` verdict (`src/trace.py:258-265`; generator:
``tests/golden/make_goldens.py replay``).  These are the vectors a native
trace replay must reproduce byte for byte.  Here they are (1) pinned against
the reference itself where it is importable, and (2) fed through the native
IR front end and instantiator, which must parse and plan every accepted
program the reference's replay produces (mutations included)."""
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
def test_fixture_shape(name):
    hdr, rows = load_replay(name)
    assert hdr["rows"] == len(rows) > 0
    kinds = {r["kind"] for r in rows}
    assert kinds == {"sampled", "mutated"}
    for r in rows:
        if r["accepted"]:
            assert r["program"] and isinstance(r["hash"], int)
        else:
            assert r["reason"] and r["index"] >= 0


@needs_reference
@pytest.mark.parametrize("name", TASKS)
def test_fixture_pinned_to_reference_validate_trace(name):
    from paper_2205_13603_b200.refapi import loopsched
    ls = loopsched()
    hdr, rows = load_replay(name)
    e0 = ls.ir.deserialize(hdr["e0"])
    for r in rows:
        t = ls.trace.deserialize_trace(r["trace"])
        v = ls.trace.validate_trace(e0, t)
        if r["accepted"]:
            assert isinstance(v, ls.trace.Accepted), r["trace"]
            assert ls.ir.serialize(v.program) == r["program"]
            assert ls.ir.structural_hash(v.program) == r["hash"]
            if "normalized" in r:
                assert ls.trace.serialize_trace(v.trace) == r["normalized"]
        else:
            assert isinstance(v, ls.trace.Rejected)
            assert (v.reason, v.index) == (r["reason"], r["index"])


@pytest.mark.parametrize("name", TASKS)
def test_native_front_end_plans_every_replayed_program(name):
    from paper_2205_13603_b200 import native
    hdr, rows = load_replay(name)
    progs = [r["program"] for r in rows if r["accepted"]]
    plans = native.plan_programs(hdr["e0"], progs)
    assert len(plans) == len(progs)
    # every replayed program parses and maps to a kernel family (ILLEGAL =
    # the hardware validator's verdict on a mapped schedule, e.g. > 1024 threads)
    bad = [p for p in plans if p["status"] not in ("OK", "ILLEGAL")]
    assert not bad, bad[:3]
    assert sum(p["status"] == "OK" for p in plans) > len(plans) // 4
