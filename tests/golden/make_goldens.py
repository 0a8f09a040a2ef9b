"""Generate the committed golden fixtures from the reference itself.

Run in a container where the reference `loopsched` is importable
(``PYTHONPATH=/root/reference/pkg/src python tests/golden/make_goldens.py``).
Everything written here is produced by the reference's own functions:

* ``programs.jsonl``   — a diverse program set with, per program, the
  reference's exact ``simulate_latency`` (`src/machine.py:228-254`), its
  ``featurize`` vector (`src/costmodel.py:21-79`) and the prediction of a model
  ``fit`` on the set (`src/costmodel.py:118-150`, `:98-102`).  Includes the
  hand-computed programs of the reference's ``tests/test_machine.py:17-184``.
* ``model.json``       — that fitted model (weights, mean, scale, intercept).
* ``pop_<task>.jsonl.gz`` — fixed populations of distinct validated programs
  per BASELINE config (the Runner's unit of work), each with
  reference latency and features.
* ``tune_<task>.json`` — reference ``tune`` reports (chosen trace, full log).
* ``outputs_small.npz`` — ``random_inputs`` + ``interp.run`` outputs at small
  shapes, pinning the numpy output oracle.
* ``replay_<task>.jsonl.gz`` — sampled traces and single-decision mutations of
  them with the reference's ``validate_trace`` verdict (`src/trace.py:258-265`):
  accepted -> the replayed program's ``ir.serialize`` text, structural hash
  and normalized trace; rejected -> reason and instruction index.  The parity
  vectors for a native trace replay.

The GPU box never runs this script (the reference does not travel there); the
fixtures do.
"""

from __future__ import annotations

import gzip
import hashlib
import json
import os
import random
import sys
from fractions import Fraction

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from paper_2205_13603_b200.refapi import loopsched  # noqa: E402
from paper_2205_13603_b200 import workloads as W, tensor_core as T  # noqa: E402

ls = loopsched()
from loopsched import ir  # noqa: E402
from loopsched.costmodel import featurize, fit, unfit_model  # noqa: E402
from loopsched.machine import MachineSpec, simulate_latency  # noqa: E402
from loopsched.schedule import ScheduleState  # noqa: E402
from loopsched.spaces import run_generator, sample_traces  # noqa: E402
from loopsched.search import SearchConfig, tune  # noqa: E402
from loopsched.trace import Accepted, mutate, serialize_trace, validate_trace  # noqa: E402

SPEC = MachineSpec()


def frac(x: Fraction):
    return [x.numerator, x.denominator]


def hand_programs():
    """The programs behind the reference's hand-computed latency tests."""
    out = []
    I = ir
    p = I.TensorProgram(
        buffers=(I.Buffer("A", (1,), "input"), I.Buffer("B", (1,), "output")),
        root=(I.Compute("c", "B", (I.IntConst(0),),
                        I.add(I.Load("A", (I.IntConst(0),)), I.IntConst(1))),))
    out.append(("hand_base_3", p))
    out.append(("hand_relu1024_3072", ls.relu1d(1024)))
    s = ScheduleState(ls.relu1d(1024))
    b, = s.get_blocks(); lp, = s.get_loops(b)
    i0, i1, i2 = s.split(lp, [32, 8, 4]); s.parallelize(i0); s.vectorize(i2)
    out.append(("hand_relu_sched_192", s.program))
    out.append(("hand_gmm4_400", ls.gmm(4, 4, 4)))
    s = ScheduleState(ls.gmm(4, 4, 4))
    b, = s.get_blocks(); loops = s.get_loops(b); s.tensorize(loops[0], "tu.mma4")
    out.append(("hand_mma4_56", s.program))
    out.append(("hand_gmm16_24832", ls.gmm(16, 16, 16)))
    out.append(("hand_gmm64_5304768", ls.gmm(64, 64, 64)))
    s = ScheduleState(ls.gmm(64, 64, 64))
    b, = s.get_blocks(); li, lj, lk = s.get_loops(b)
    i0, i1 = s.split(li, [8, 8]); j0, j1 = s.split(lj, [8, 8]); k0, k1 = s.split(lk, [8, 8])
    s.reorder([i0, j0, k0, i1, j1, k1])
    out.append(("hand_gmm64_tiled", s.program))
    tp = I.TensorProgram(
        buffers=(I.Buffer("A", (16, 16), "input"), I.Buffer("B", (16, 16), "output")),
        root=(I.Loop("i", 16, "serial", (I.Loop("j", 16, "serial", (
            I.Compute("t", "B", (I.var("i"), I.var("j")),
                      I.load("A", I.var("j"), I.var("i"))),)),)),))
    s = ScheduleState(tp); blk, = s.get_blocks(); _, lj = s.get_loops(blk); s.vectorize(lj)
    out.append(("hand_transpose_vec_nodiscount", s.program))
    q = I.TensorProgram(
        buffers=(I.Buffer("A", (16, 16), "input"), I.Buffer("B", (16, 16), "output")),
        root=(I.Loop("i", 16, "serial", (I.Loop("j", 16, "serial", (
            I.Compute("t", "B", (I.var("i"), I.var("j")),
                      I.load("A", I.var("i"), I.var("j"))),)),)),))
    out.append(("hand_copy_512", q))
    s = ScheduleState(q); blk, = s.get_blocks(); _, lj = s.get_loops(blk); s.vectorize(lj)
    out.append(("hand_copy_vec_64", s.program))
    s = ScheduleState(ls.relu1d(64)); b, = s.get_blocks(); lp, = s.get_loops(b)
    o, i = s.split(lp, [16, 4]); s.parallelize(o); s.parallelize(i)
    out.append(("hand_nested_parallel", s.program))
    s = ScheduleState(ls.relu1d(64)); b, = s.get_blocks(); lp, = s.get_loops(b)
    o, i = s.split(lp, [4, 16]); s.unroll(i)
    out.append(("hand_unroll16_discount", s.program))
    s = ScheduleState(ls.relu1d(64)); b, = s.get_blocks(); lp, = s.get_loops(b)
    o, i = s.split(lp, [2, 32]); s.unroll(i)
    out.append(("hand_unroll32_nodiscount", s.program))
    s = ScheduleState(ls.gmm(8, 8, 8)); b, = s.get_blocks(); li, lj, lk = s.get_loops(b)
    i0, i1 = s.split(li, [2, 4]); j0, j1 = s.split(lj, [2, 4]); k0, k1 = s.split(lk, [2, 4])
    s.reorder([i0, j0, k0, i1, j1, k1]); s.tensorize(i1, "tu.mma4")
    out.append(("hand_tensor_calls_8", s.program))
    return out


SMALL = [lambda: ls.relu1d(48), lambda: ls.gmm(8, 8, 8), lambda: ls.gmm(12, 6, 4),
         lambda: ls.dense_relu(8, 8, 8), lambda: ls.conv1d(12, 2, 3, 3, 1, 1),
         lambda: W.batch_matmul(2, 8, 8, 4), lambda: W.conv2d_nhwc(1, 6, 6, 2, 3, 3, 3, 1, 1)]


def random_programs(n: int, seed: int):
    rng = random.Random(seed)
    spaces = [ls.default_space(),
              T.space_from_config({"modules": [{"mlt": {"structure": "SSRSR"}},
                                               {"auto_inline": {}},
                                               {"pvu": {"widths": [4, 8]}},
                                               {"tensor_unit": {}}]})]
    out = []
    for i in range(n):
        e0 = SMALL[rng.randrange(len(SMALL))]()
        gen = spaces[rng.randrange(len(spaces))]
        prog, _ = run_generator(e0, gen, rng.randrange(2 ** 62))
        out.append((f"random_{i}", prog))
    return out


def big_programs():
    """Programs at the BASELINE config shapes."""
    out = []
    tasks = [("gmm512", ls.gmm(512, 512, 512), ls.default_space()),
             ("bert_ffn", ls.gmm(128, 768, 3072), T.b200_space()),
             ("bmm_qk", W.batch_matmul(12, 128, 128, 64), T.b200_space()),
             ("conv2d", W.conv2d_nhwc(), ls.default_space()),
             ("dense_relu", ls.dense_relu(128, 128, 128), T.b200_space())]
    for name, e0, gen in tasks:
        out.append((f"{name}_e0", e0))
        for j, (prog, _) in enumerate(sample_traces(e0, gen, 12, seed=7)):
            out.append((f"{name}_s{j}", prog))
    return out


def write_programs():
    items = hand_programs() + random_programs(160, seed=11) + big_programs()
    rows = []
    for name, p in items:
        lat = simulate_latency(p, SPEC)
        f = featurize(p, SPEC)
        rows.append({"name": name, "program": ir.serialize(p),
                     "hash": ir.structural_hash(p), "latency": frac(lat),
                     "features": [float(x) for x in f]})
    model = fit(unfit_model(), [(np.array(r["features"]), Fraction(*r["latency"]))
                                for r in rows])
    for r in rows:
        r["predicted"] = model.predict_features(np.array(r["features"]))
    with open(os.path.join(HERE, "programs.jsonl"), "w") as fh:
        for r in rows:
            fh.write(json.dumps(r, sort_keys=True) + "\n")
    with open(os.path.join(HERE, "model.json"), "w") as fh:
        json.dump({"weights": list(map(float, model.weights)),
                   "feature_mean": list(map(float, model.feature_mean)),
                   "feature_scale": list(map(float, model.feature_scale)),
                   "intercept": float(model.intercept), "n_records": model.n_records,
                   "degenerate": bool(model.degenerate)}, fh, indent=1, sort_keys=True)
    print("programs", len(rows))


POPULATIONS = {
    # name: (builder, space-config, size); 8192 = 8 GPUs x 1024 distinct
    # candidates per rank for the four bench workloads (disjoint rank slices
    # at every N), 1024 for the other config-5 tasks
    "bert_ffn": (lambda: ls.gmm(128, 768, 3072), T.b200_space_config(), 8192),
    "bmm_qk": (lambda: W.batch_matmul(12, 128, 128, 64), T.b200_space_config(), 8192),
    "gmm512": (lambda: ls.gmm(512, 512, 512), ls.default_space_config(), 8192),
    # config 1 with the tcgen05 module: fp32 tiles run as 3xTF32
    "gmm512_tc": (lambda: ls.gmm(512, 512, 512), T.b200_space_config(), 8192),
    "conv2d": (lambda: W.conv2d_nhwc(), T.b200_space_config(), 8192),
    "bert_dense": (lambda: ls.gmm(128, 768, 768), T.b200_space_config(), 1024),
    "bert_ffn_in": (lambda: ls.gmm(128, 3072, 768), T.b200_space_config(), 1024),
    "bmm_pv": (lambda: W.batch_matmul(12, 128, 64, 128), T.b200_space_config(), 1024),
}


def write_population(name: str):
    build, space_doc, size = POPULATIONS[name]
    e0 = build()
    gen = T.space_from_config(space_doc)
    rng = random.Random(2022)
    seen = {}
    attempts = 0
    while len(seen) < size and attempts < 40 * size:
        attempts += 1
        prog, _ = run_generator(e0, gen, rng.randrange(2 ** 62))
        h = ir.structural_hash(prog)
        if h not in seen:
            seen[h] = prog
    path = os.path.join(HERE, f"pop_{name}.jsonl.gz")
    with gzip.open(path, "wt") as fh:
        fh.write(json.dumps({"workload": name, "e0": ir.serialize(e0),
                             "space": space_doc, "seed": 2022, "size": len(seen),
                             "machine_spec": SPEC.to_json()}, sort_keys=True) + "\n")
        for h, p in seen.items():
            fh.write(json.dumps({"hash": h, "program": ir.serialize(p),
                                 "latency": frac(simulate_latency(p, SPEC)),
                                 "features": [float(x) for x in featurize(p, SPEC)]},
                                sort_keys=True) + "\n")
    print("population", name, len(seen), "attempts", attempts)


def write_replay(name: str, samples: int = 48, mutations: int = 3):
    build, space_doc, _ = POPULATIONS[name]
    e0 = build()
    gen = T.space_from_config(space_doc)
    rng = random.Random(2205)
    rows = []
    for _ in range(samples):
        prog, trace = run_generator(e0, gen, rng.randrange(2 ** 62))
        rows.append({"kind": "sampled", "trace": serialize_trace(trace), "accepted": True,
                     "program": ir.serialize(prog), "hash": ir.structural_hash(prog)})
        for _ in range(mutations):
            t2, pos = mutate(trace, rng)
            if pos is None:
                continue
            v = validate_trace(e0, t2)
            row = {"kind": "mutated", "mutated_index": pos, "trace": serialize_trace(t2),
                   "accepted": isinstance(v, Accepted)}
            if isinstance(v, Accepted):
                row.update(program=ir.serialize(v.program), hash=ir.structural_hash(v.program),
                           normalized=serialize_trace(v.trace))
            else:
                row.update(reason=v.reason, index=v.index)
            rows.append(row)
    path = os.path.join(HERE, f"replay_{name}.jsonl.gz")
    with gzip.open(path, "wt") as fh:
        fh.write(json.dumps({"workload": name, "e0": ir.serialize(e0), "space": space_doc,
                             "seed": 2205, "rows": len(rows)}, sort_keys=True) + "\n")
        for r in rows:
            fh.write(json.dumps(r, sort_keys=True) + "\n")
    print("replay", name, len(rows), "accepted", sum(r["accepted"] for r in rows))


def write_tune(name: str, e0, space_doc, trials: int, seed: int):
    report = tune(e0, T.space_from_config(space_doc),
                  SearchConfig(trials=trials, seed=seed), SPEC)
    doc = report.to_json(timestamp=False)
    doc["sha256"] = hashlib.sha256(json.dumps(doc, sort_keys=True).encode()).hexdigest()
    doc["e0"] = ir.serialize(e0)
    doc["log_programs"] = []
    # programs of every logged record (replayed from their traces)
    from loopsched.trace import validate_trace
    for rec in report.log:
        v = validate_trace(e0, rec.trace)
        doc["log_programs"].append(ir.serialize(v.program))
    with open(os.path.join(HERE, f"tune_{name}.json"), "w") as fh:
        json.dump(doc, fh, sort_keys=True)
    print("tune", name, doc["best"]["latency"], doc["sha256"][:16])


def write_outputs():
    from loopsched import interp
    arrays = {}
    cases = {"gmm": ls.gmm(16, 12, 20), "bmm": W.batch_matmul(3, 8, 12, 16),
             "conv2d": W.conv2d_nhwc(1, 6, 5, 3, 4, 3, 3, 1, 1),
             "dense_relu": ls.dense_relu(8, 12, 16)}
    for name, e0 in cases.items():
        for seed in (0, 1):
            inp = interp.random_inputs(e0, seed)
            out = interp.run(e0, inp)
            for k, v in inp.items():
                arrays[f"{name}/s{seed}/in/{k}"] = v.as_array()
            for k, v in out.items():
                arrays[f"{name}/s{seed}/out/{k}"] = v.as_array()
        arrays[f"{name}/e0"] = np.frombuffer(ir.serialize(e0).encode(), dtype=np.uint8)
    np.savez_compressed(os.path.join(HERE, "outputs_small.npz"), **arrays)
    print("outputs", len(arrays))


BIG_OUTPUT_CASES = {
    # the BASELINE config shapes incl. every config-5 task
    "gmm512": lambda: ls.gmm(512, 512, 512),
    "bert_ffn": lambda: ls.gmm(128, 768, 3072),
    "bert_dense": lambda: ls.gmm(128, 768, 768),
    "bert_ffn_in": lambda: ls.gmm(128, 3072, 768),
    "bmm_qk": lambda: W.batch_matmul(12, 128, 128, 64),
    "bmm_pv": lambda: W.batch_matmul(12, 128, 64, 128),
    "conv2d": lambda: W.conv2d_nhwc(),
}


def write_outputs_big():
    """sha256 of the reference interpreter's own inputs and outputs
    (`interp.random_inputs(e0, 0)`, `interp.run`, `src/interp.py:54-63`,
    `:314-342`) at the full BASELINE shapes, as int64 C-order bytes: pins the
    numpy output oracle (oracle.reference_outputs) and the repo's
    random_inputs at the sizes the GPU parity tests run."""
    from loopsched import interp
    doc = {}
    for name, build in BIG_OUTPUT_CASES.items():
        e0 = build()
        inp = interp.random_inputs(e0, 0)
        out = interp.run(e0, inp)
        sha = lambda a: hashlib.sha256(np.ascontiguousarray(a, dtype=np.int64).tobytes()).hexdigest()
        doc[name] = {"e0": ir.serialize(e0), "seed": 0,
                     "inputs": {k: sha(v.as_array()) for k, v in inp.items()},
                     "outputs": {k: {"sha256": sha(v.as_array()), "shape": list(v.as_array().shape),
                                     "max_abs": int(np.abs(v.as_array()).max())} for k, v in out.items()}}
        print("outputs_big", name, {k: v["max_abs"] for k, v in doc[name]["outputs"].items()})
    with open(os.path.join(HERE, "outputs_big.json"), "w") as fh:
        json.dump(doc, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    what = sys.argv[1:] or ["programs", "pops", "tune", "outputs"]
    if "programs" in what:
        write_programs()
    if "pops" in what:
        for n in POPULATIONS:
            write_population(n)
    for n in POPULATIONS:
        if f"pop:{n}" in what:
            write_population(n)
    if "tune" in what:
        write_tune("gmm512", ls.gmm(512, 512, 512), ls.default_space_config(), 64, 0)
        write_tune("gmm512_tu", ls.gmm(512, 512, 512),
                   {"modules": ls.default_space_config()["modules"] + [{"tensor_unit": {}}]},
                   64, 0)
        write_tune("bert_ffn", ls.gmm(128, 768, 3072), T.b200_space_config(), 64, 0)
    if "outputs" in what:
        write_outputs()
    if "outputs_big" in what:
        write_outputs_big()
    if "replay" in what:
        for n in POPULATIONS:
            write_replay(n)
