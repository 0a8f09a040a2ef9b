"""Search-side pieces that need the reference package (skipped without it):
the tcgen05 tiling module, the new workload builders and the input mirror."""
import json
import random

import numpy as np
import pytest

from conftest import needs_reference

pytestmark = needs_reference


@pytest.fixture(scope="module")
def ls():
    from paper_2205_13603_b200.refapi import loopsched
    return loopsched()


def test_random_inputs_mirror_reference(ls):
    from paper_2205_13603_b200.inputs import random_inputs
    from paper_2205_13603_b200.workloads import batch_matmul
    for e0 in (ls.gmm(16, 12, 20), batch_matmul(2, 8, 8, 4), ls.dense_relu(8, 8, 8)):
        ref = ls.random_inputs(e0, 3)
        mine = random_inputs(ls.ir.serialize(e0), 3)
        assert set(ref) == set(mine)
        for k in ref:
            assert np.array_equal(ref[k].as_array(), mine[k])


def test_builders_valid_and_schedulable(ls):
    from paper_2205_13603_b200.workloads import batch_matmul, conv2d_nhwc
    from loopsched.spaces import run_generator
    rng = random.Random(0)
    for e0 in (batch_matmul(2, 8, 8, 4), conv2d_nhwc(1, 5, 6, 2, 3, 3, 3, 1, 1),
               conv2d_nhwc(1, 7, 7, 2, 2, 3, 3, 2, 1)):
        refs = {s: ls.run(e0, ls.random_inputs(e0, s)) for s in (0, 1)}
        for _ in range(15):
            prog, trace = run_generator(e0, ls.default_space(), rng.randrange(2 ** 62))
            for s in (0, 1):
                assert ls.outputs_equal(ls.run(prog, ls.random_inputs(e0, s)), refs[s])


def test_conv2d_matches_direct_convolution(ls):
    from paper_2205_13603_b200.workloads import conv2d_nhwc
    e0 = conv2d_nhwc(1, 6, 5, 3, 4, 3, 3, 1, 1)
    inp = ls.random_inputs(e0, 0)
    X, W = inp["X"].as_array(), inp["W"].as_array()
    Xp = np.pad(X, ((0, 0), (1, 1), (1, 1), (0, 0)))
    O = np.zeros((1, 6, 5, 4), dtype=np.int64)
    for r in range(3):
        for s in range(3):
            O += Xp[:, r:r + 6, s:s + 5, :] @ W[r, s]
    assert np.array_equal(ls.run(e0, inp)["O"].as_array(), O)


def test_tensor_core_module_semantics_and_replay(ls):
    from paper_2205_13603_b200 import tensor_core as T
    from paper_2205_13603_b200.workloads import batch_matmul
    from loopsched.spaces import run_generator
    from loopsched.trace import mutate, validate_trace
    gen = ls.compose([T.use_tensor_core()])
    rng = random.Random(1)
    for e0 in (ls.gmm(128, 48, 128), batch_matmul(2, 128, 32, 64)):
        ref = ls.run(e0, ls.random_inputs(e0, 0))
        for _ in range(6):
            prog, trace = run_generator(e0, gen, rng.randrange(2 ** 62))
            assert any(i.op == "reorder" for i in trace.instructions)
            assert ls.outputs_equal(ls.run(prog, ls.random_inputs(e0, 0)), ref)
            v = validate_trace(e0, trace)
            assert ls.structural_equal(v.program, prog)
            t2, pos = mutate(trace, rng)
            if pos is not None:
                v2 = validate_trace(e0, t2)
                if isinstance(v2, ls.Accepted):
                    assert ls.outputs_equal(ls.run(v2.program, ls.random_inputs(e0, 0)), ref)


def test_tensor_core_module_applicability(ls):
    from paper_2205_13603_b200 import tensor_core as T
    from paper_2205_13603_b200.workloads import conv2d_nhwc
    from loopsched.schedule import ScheduleState
    mod = T.use_tensor_core()
    for e0, want in ((ls.gmm(128, 768, 3072), True), (ls.gmm(64, 64, 64), False),
                     (ls.relu1d(64), False), (conv2d_nhwc(1, 6, 6, 2, 3, 3, 3, 1, 1), False)):
        s = ScheduleState(e0)
        blocks = s.get_blocks()
        assert any(mod.applicability(s, b) for b in blocks) == want


def test_tensor_core_programs_map_to_tcgen05(ls):
    from paper_2205_13603_b200 import native, tensor_core as T
    from loopsched.spaces import sample_traces
    e0 = ls.gmm(128, 768, 3072)
    progs = [ls.ir.serialize(p) for p, _ in sample_traces(e0, ls.compose([T.use_tensor_core()]), 20, seed=3)]
    res = native.plan_programs(ls.ir.serialize(e0), progs, "bf16")
    for r in res:
        assert r["family"] == "tcgen05"
        assert r["status"] == ("OK" if r["cfg"][3] <= 256 else "ILLEGAL")
