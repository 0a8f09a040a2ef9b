"""Workload inputs and program text helpers.

``random_inputs`` reproduces the reference's input generator
(`src/interp.py:54-63`: numpy PCG64 ``default_rng(seed)``, integers in
[-8, 8], one draw per input buffer in declaration order) from the program's
JSON text alone, so the GPU box needs no reference install to build the exact
tensors the reference interpreter would see.
"""

from __future__ import annotations

import json

import numpy as np

from .refapi import loopsched


def program_text(p) -> str:
    """JSON text of a program: passes strings through, serializes reference
    ``TensorProgram`` objects with the reference's own ``ir.serialize``."""
    if isinstance(p, str):
        return p
    if isinstance(p, (bytes, bytearray)):
        return p.decode()
    prog = getattr(p, "program", p)  # a search Candidate / TuningRecord-like object
    if isinstance(prog, str):
        return prog
    text = getattr(prog, "_ls_text", None)  # replay.LazyProgram: the native replay's own text
    if text is not None:
        return text
    return loopsched().ir.serialize(prog)


def input_buffers(e0_json: str):
    doc = json.loads(e0_json)
    return [(b["name"], tuple(b["shape"])) for b in doc["buffers"] if b["role"] == "input"]


def random_inputs(e0_json: str, seed: int) -> dict:
    rng = np.random.default_rng(seed)
    return {name: rng.integers(-8, 9, size=shape, dtype=np.int64)
            for name, shape in input_buffers(e0_json)}


def normal_inputs(e0_json: str, seed: int) -> dict:
    """N(0,1) float inputs for the floating-point tolerance checks."""
    rng = np.random.default_rng(seed)
    return {name: rng.standard_normal(size=shape) for name, shape in input_buffers(e0_json)}


def output_buffers(e0_json: str):
    doc = json.loads(e0_json)
    return [(b["name"], tuple(b["shape"])) for b in doc["buffers"] if b["role"] == "output"]
