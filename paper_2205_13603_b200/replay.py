"""Native trace replay behind the reference's validator.

``validate_trace`` (`src/trace.py:258-265`) -- a Python replay of every
schedule primitive (`src/schedule.py:123-974`) -- is what caps the
reference's search once measurement and scoring run on the GPU.  This module
routes it through ``ls_replay_batch`` (csrc/replay.cpp), which restates the
replay natively and returns the reference's exact outputs: the accepted
program's ``ir.serialize`` text and ``ir.structural_hash``, the normalized
trace's ``serialize_trace`` text, or the (reason, index) of a rejection.

``NativeValidator`` subclasses the reference's own ``_Validator``
(`src/search.py:100-146`) and overrides only ``candidate``; the cache, the
feature memo, ``_revive`` and the ``_predict`` seam are the reference's.  The
program of an accepted candidate is a ``LazyProgram``: it carries the
serialized text (what the B200 seams consume) and materializes the reference
``TensorProgram`` only if something asks for its tree.

Traces the native replay defers (inputs on which the reference would raise
something other than ``ReplayError``) are validated by the reference itself,
so behaviour is identical by construction.
"""

from __future__ import annotations

import ctypes
import dataclasses
import json

from . import native
from .refapi import loopsched

ACCEPTED, REJECTED, DEFER = 0, 1, 2


class NativeReplayer:
    """One workload; ``validate(keys)`` replays a batch of serialized traces."""

    def __init__(self, e0_text: str):
        L = native.lib()
        h = ctypes.c_void_p()
        e = e0_text.encode()
        native.check(L.ls_replayer_create(e, len(e), ctypes.byref(h)), "ls_replayer_create")
        self._h = h
        self._L = L
        v = ctypes.c_uint64()
        native.check(L.ls_replayer_hash(h, ctypes.byref(v)), "ls_replayer_hash")
        self.workload_hash = v.value

    def validate(self, keys):
        """[(status, index, hash, program_text, trace_text, reason)] per key."""
        n = len(keys)
        if n == 0:
            return []
        arr, lens, _keep = native.text_array(keys)
        res = (native.ReplayResultC * n)()
        native.check(self._L.ls_replay_batch(self._h, arr, lens, n, res), "ls_replay_batch")
        out = []
        sa = ctypes.string_at
        for r in res:
            st = r.status
            if st == ACCEPTED:
                out.append((st, r.index, r.hash, sa(r.program).decode(), sa(r.trace).decode(), None))
            else:
                out.append((st, r.index, 0, None, None, sa(r.reason).decode() if r.reason else ""))
        self._L.ls_replay_free(res, n)
        return out

    def close(self):
        if self._h:
            self._L.ls_replayer_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def program_hash(text: str) -> int:
    """``ir.structural_hash`` of a serialized program (`src/ir.py:625-629`)."""
    v = ctypes.c_uint64()
    b = text.encode()
    native.check(native.lib().ls_program_hash(b, len(b), ctypes.byref(v)), "ls_program_hash")
    return v.value


_LAZY = None


def lazy_program_class():
    """A ``TensorProgram`` (`src/ir.py:160-175`) backed by its serialized text;
    the tree is deserialized on first access to ``buffers`` / ``root``."""
    global _LAZY
    if _LAZY is None:
        ir = loopsched().ir

        class LazyProgram(ir.TensorProgram):
            def __init__(self, text: str):  # noqa: D107 -- the frozen fields are properties here
                object.__setattr__(self, "_ls_text", text)
                object.__setattr__(self, "_ls_tree", None)

            def _tree(self):
                t = self._ls_tree
                if t is None:
                    t = ir.deserialize(self._ls_text)
                    object.__setattr__(self, "_ls_tree", t)
                return t

            @property
            def buffers(self):
                return self._tree().buffers

            @property
            def root(self):
                return self._tree().root

            def __eq__(self, other):  # equal to the reference object it stands for
                if isinstance(other, ir.TensorProgram):
                    return (self.buffers, self.root) == (other.buffers, other.root)
                return NotImplemented

            def __hash__(self):
                return hash((self.buffers, self.root))

        _LAZY = LazyProgram
    return _LAZY


def normalized_trace(key: str, text: str, t):
    """The reference's normalized trace (`src/trace.py:196-198`) from the
    native ``serialize_trace`` text, reusing the input's instruction objects
    wherever the line is unchanged."""
    tr = loopsched().trace
    if text == key:
        return dataclasses.replace(t, validated=True)
    old = key.splitlines()
    new = text.splitlines()
    off_old = 1 if t.workload_hash is not None else 0
    ins = []
    for k, line in enumerate(new[off_old:]):
        j = k + off_old
        if j < len(old) and old[j] == line:
            ins.append(t.instructions[k])
        else:
            d = json.loads(line)
            ins.append(tr.Instruction(d["op"], tuple(d.get("inputs", [])), d.get("attrs", {}),
                                      tuple(d.get("outputs", [])), d.get("decision")))
    return tr.Trace(tuple(ins), workload_hash=t.workload_hash, validated=True)


_NATIVE_VALIDATOR = None


def native_validator_class():
    """``_Validator`` (`src/search.py:100-146`) with ``candidate`` replayed natively."""
    global _NATIVE_VALIDATOR
    if _NATIVE_VALIDATOR is None:
        ls = loopsched()
        S = ls.search
        base = S._Validator._ls_base if getattr(S._Validator, "_ls_dispatch", False) else S._Validator

        class NativeValidator(base):
            def __init__(self, e0, machine_spec=None):
                if machine_spec is None:
                    super().__init__(e0, ls.MachineSpec())
                else:
                    super().__init__(e0, machine_spec)
                self._rp = NativeReplayer(ls.ir.serialize(e0))
                self._lazy = lazy_program_class()
                self.native_calls = 0
                self.deferred = 0

            def candidate(self, t, model):
                key = ls.trace.serialize_trace(t)
                if key in self.cache:
                    return self._revive(self.cache[key], model)
                (st, _idx, h, prog, norm, _reason), = self._rp.validate([key])
                self.native_calls += 1
                if st == REJECTED:
                    self.cache[key] = None
                    return None
                if st == DEFER:
                    self.deferred += 1
                    return base.candidate(self, t, model)
                return self._store_native(key, normalized_trace(key, norm, t), self._lazy(prog), h, model)

            def prevalidate(self, traces):
                """Validate a batch of traces in one native call and store the
                accepted/rejected verdicts, so the sequential ``candidate``
                calls that follow are cache hits (featurize stays per program)."""
                keys, seen = [], set()
                for t in traces:
                    k = ls.trace.serialize_trace(t)
                    if k not in self.cache and k not in seen:
                        seen.add(k)
                        keys.append((k, t))
                out = self._rp.validate([k for k, _ in keys])
                self.native_calls += len(keys)
                ready = []
                for (k, t), (st, _idx, h, prog, norm, _r) in zip(keys, out):
                    if st == REJECTED:
                        self.cache[k] = None
                    elif st == ACCEPTED:
                        ready.append((k, normalized_trace(k, norm, t), self._lazy(prog), h))
                return ready

            def _store_native(self, key, t, program, h, model):
                # _Validator._store (`src/search.py:137-146`) with the hash the
                # native replay computed
                feats = self.features_by_hash.get(h)
                if feats is None:
                    feats = S.featurize(program, self.machine_spec)
                    self.features_by_hash[h] = feats
                cand = S.Candidate(t, program, h, feats, self._predict(program, feats, model))
                self.cache[key] = cand
                return cand

        _NATIVE_VALIDATOR = NativeValidator
    return _NATIVE_VALIDATOR
