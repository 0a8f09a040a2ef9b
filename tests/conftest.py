"""Shared test setup: markers, paths, golden loaders."""
import gzip
import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs under gpurun)")


def load_programs():
    with open(os.path.join(GOLDEN, "programs.jsonl")) as fh:
        return [json.loads(l) for l in fh]


def load_model():
    with open(os.path.join(GOLDEN, "model.json")) as fh:
        return json.load(fh)


def load_population(name):
    with gzip.open(os.path.join(GOLDEN, f"pop_{name}.jsonl.gz"), "rt") as fh:
        lines = fh.read().splitlines()
    return json.loads(lines[0]), [json.loads(l) for l in lines[1:]]


def has_reference():
    try:
        from paper_2205_13603_b200.refapi import loopsched
        loopsched()
        return True
    except ImportError:
        return False


needs_reference = pytest.mark.skipif(not has_reference(),
                                     reason="reference loopsched not importable here")
