"""TEST INFRASTRUCTURE ONLY — the CPU oracle (parity checker + CPU baseline).

Python face of ``ls_oracle.c`` (a C restatement of the reference's
``simulate_latency`` / ``featurize`` / ``predict_features``) plus a numpy
restatement of the reference interpreter's output semantics for the workload
families on the measured path (``src/interp.py:314-342``; exact int64 values
through float64 products, which are exact below 2**53).

Import rules: only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this module.  The
product package never does.

Parity pinning: ``tests/test_oracle.py`` checks every function here against
the reference's own outputs committed under ``tests/golden/``.
"""

from __future__ import annotations

import ctypes
import json
import os
import subprocess
from fractions import Fraction

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "build", "libls_oracle.so")


class Spec(ctypes.Structure):
    _fields_ = [(n, ctypes.c_longlong) for n in
                ("cores", "vector_lanes", "cache_capacity", "hit_cost", "miss_cost",
                 "flop_cost", "tensor_unit_cost", "unroll_num", "unroll_den")]


class Model(ctypes.Structure):
    _fields_ = [("w", ctypes.c_double * 9), ("mean", ctypes.c_double * 9),
                ("scale", ctypes.c_double * 9), ("intercept", ctypes.c_double),
                ("n_records", ctypes.c_longlong), ("is_fit", ctypes.c_int)]


DEFAULT_SPEC = {"cores": 4, "vector_lanes": 8, "cache_capacity": 4096, "hit_cost": 1,
                "miss_cost": 8, "flop_cost": 1, "unroll_discount": 0.9,
                "tensor_unit_cost": 8}


def build() -> str:
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = ctypes.CDLL(LIB_PATH)
        L.lso_sim_latency.argtypes = [ctypes.c_char_p, ctypes.c_long, ctypes.POINTER(Spec),
                                      ctypes.POINTER(ctypes.c_longlong),
                                      ctypes.POINTER(ctypes.c_longlong)]
        L.lso_featurize.argtypes = [ctypes.c_char_p, ctypes.c_long, ctypes.POINTER(Spec),
                                    ctypes.POINTER(ctypes.c_double)]
        L.lso_predict.argtypes = [ctypes.POINTER(ctypes.c_double), ctypes.POINTER(Model)]
        L.lso_predict.restype = ctypes.c_double
        L.lso_batch.argtypes = [ctypes.POINTER(ctypes.c_char_p), ctypes.POINTER(ctypes.c_long),
                                ctypes.c_int, ctypes.POINTER(Spec), ctypes.POINTER(Model),
                                ctypes.c_int, ctypes.POINTER(ctypes.c_longlong),
                                ctypes.POINTER(ctypes.c_longlong),
                                ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double),
                                ctypes.POINTER(ctypes.c_int)]
        _lib = L
    return _lib


def make_spec(doc=None) -> Spec:
    d = dict(DEFAULT_SPEC)
    d.update(doc or {})
    disc = Fraction(str(d["unroll_discount"]))
    return Spec(d["cores"], d["vector_lanes"], d["cache_capacity"], d["hit_cost"],
                d["miss_cost"], d["flop_cost"], d["tensor_unit_cost"],
                disc.numerator, disc.denominator)


def make_model(doc) -> Model:
    """doc: {'weights','feature_mean','feature_scale','intercept','n_records'} or
    weights None for an unfit model."""
    m = Model()
    w = doc.get("weights")
    m.is_fit = 1 if w is not None else 0
    if w is not None:
        for i in range(9):
            m.w[i] = w[i]
            m.mean[i] = doc["feature_mean"][i]
            m.scale[i] = doc["feature_scale"][i]
    m.intercept = doc.get("intercept", 0.0)
    m.n_records = doc.get("n_records", 0)
    return m


def sim_latency(program_json: str, spec=None) -> Fraction:
    b = program_json.encode()
    num, den = ctypes.c_longlong(), ctypes.c_longlong()
    st = lib().lso_sim_latency(b, len(b), ctypes.byref(make_spec(spec)),
                               ctypes.byref(num), ctypes.byref(den))
    if st:
        raise ValueError(f"oracle sim_latency status {st}")
    return Fraction(num.value, den.value)


def featurize(program_json: str, spec=None) -> np.ndarray:
    b = program_json.encode()
    out = (ctypes.c_double * 9)()
    st = lib().lso_featurize(b, len(b), ctypes.byref(make_spec(spec)), out)
    if st:
        raise ValueError(f"oracle featurize status {st}")
    return np.array(out[:], dtype=np.float64)


def predict(features, model_doc) -> float:
    f = (ctypes.c_double * 9)(*[float(x) for x in features])
    return lib().lso_predict(f, ctypes.byref(make_model(model_doc)))


def batch(programs, spec=None, model_doc=None, threads: int = 1):
    """(latency (num, den) arrays, features [n,9], predictions [n], status [n])
    for a population, on ``threads`` host threads."""
    n = len(programs)
    enc = [p.encode() for p in programs]
    texts = (ctypes.c_char_p * n)(*enc)
    lens = (ctypes.c_long * n)(*[len(b) for b in enc])
    num = np.zeros(n, np.int64)
    den = np.zeros(n, np.int64)
    feats = np.zeros((n, 9), np.float64)
    pred = np.zeros(n, np.float64)
    status = np.zeros(n, np.int32)
    P = ctypes.POINTER
    model = ctypes.byref(make_model(model_doc)) if model_doc is not None else None
    lib().lso_batch(texts, lens, n, ctypes.byref(make_spec(spec)), model, threads,
                    num.ctypes.data_as(P(ctypes.c_longlong)),
                    den.ctypes.data_as(P(ctypes.c_longlong)),
                    feats.ctypes.data_as(P(ctypes.c_double)),
                    pred.ctypes.data_as(P(ctypes.c_double)),
                    status.ctypes.data_as(P(ctypes.c_int)))
    return num, den, feats, pred, status


# ---------------------------------------------------------------------------
# output oracle (exact values of the unscheduled workload)
# ---------------------------------------------------------------------------

def workload_kind(e0_json: str) -> str:
    doc = json.loads(e0_json)
    names = [b["name"] for b in doc["buffers"]]
    if names == ["A", "B", "C"]:
        return "bmm" if len(doc["buffers"][0]["shape"]) == 3 else "gmm"
    if names == ["A", "W", "D", "R"]:
        return "dense_relu"
    if names[:2] == ["X", "W"] and names[-1] == "O" and len(doc["buffers"][0]["shape"]) == 4:
        return "conv2d"
    raise ValueError(f"no output oracle for buffers {names}")


def _conv_pad(e0_json: str) -> int:
    doc = json.loads(e0_json)
    shapes = {b["name"]: b["shape"] for b in doc["buffers"]}
    if "P" in shapes:
        return (shapes["P"][1] - shapes["X"][1]) // 2
    return 0


def reference_outputs(e0_json: str, inputs: dict) -> dict:
    """Exact outputs of the unscheduled workload on the given inputs (any
    numeric dtype; computed in float64, exact for the integer inputs the
    parity tests use)."""
    kind = workload_kind(e0_json)
    f = {k: np.asarray(v, dtype=np.float64) for k, v in inputs.items()}
    if kind == "gmm":
        return {"C": f["A"] @ f["B"]}
    if kind == "dense_relu":
        return {"R": np.maximum(f["A"] @ f["W"], 0.0)}
    if kind == "bmm":
        return {"C": np.einsum("bik,bjk->bij", f["A"], f["B"])}
    # conv2d NHWC / HWIO with stride inferred from the output shape
    doc = json.loads(e0_json)
    shapes = {b["name"]: b["shape"] for b in doc["buffers"]}
    pad = _conv_pad(e0_json)
    X, Wt = f["X"], f["W"]
    n, h, w, ci = X.shape
    r, s, _, co = Wt.shape
    _, oh, ow, _ = shapes["O"]
    stride = (h + 2 * pad - r) // (oh - 1) if oh > 1 else 1
    Xp = np.zeros((n, h + 2 * pad, w + 2 * pad, ci))
    Xp[:, pad:pad + h, pad:pad + w, :] = X
    O = np.zeros((n, oh, ow, co))
    for rr in range(r):
        for ss in range(s):
            win = Xp[:, rr:rr + stride * (oh - 1) + 1:stride, ss:ss + stride * (ow - 1) + 1:stride, :]
            O += win @ Wt[rr, ss]
    return {"O": O}
