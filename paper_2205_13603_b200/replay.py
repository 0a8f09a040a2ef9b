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

    def resample(self, key: str, seed: int):
        """``replay(e0, t, mode="resample", seed)`` of a serialized trace:
        (status, index, hash, program_text, trace_text, reason)."""
        res = native.ReplayResultC()
        b = key.encode()
        native.check(self._L.ls_replay_resample(self._h, b, len(b), seed, ctypes.byref(res)), "ls_replay_resample")
        sa = ctypes.string_at
        if res.status == ACCEPTED:
            out = (res.status, res.index, res.hash, sa(res.program).decode(), sa(res.trace).decode(), None)
        else:
            out = (res.status, res.index, 0, None, None, sa(res.reason).decode() if res.reason else "")
        self._L.ls_replay_free(ctypes.byref(res), 1)
        return out

    def neighbours(self, member_keys):
        """Replay every single-decision neighbour of each member key not
        expanded before; returns ([(hash, program_text)] for structural
        hashes not handed out before, stats dict)."""
        n = len(member_keys)
        if n == 0:
            return [], {"replayed": 0, "accepted": 0, "rejected": 0, "deferred": 0}
        arr, lens, _keep = native.text_array(member_keys)
        h = ctypes.c_void_p()
        native.check(self._L.ls_replay_neighbours(self._h, arr, lens, n, ctypes.byref(h)), "ls_replay_neighbours")
        try:
            cnt = ctypes.c_int()
            native.check(self._L.ls_neighbours_count(h, ctypes.byref(cnt)), "ls_neighbours_count")
            st = (ctypes.c_int64 * 4)()
            native.check(self._L.ls_neighbours_stats(h, st), "ls_neighbours_stats")
            hv, pg = ctypes.c_uint64(), ctypes.c_char_p()
            get = self._L.ls_neighbours_get
            out = []
            for i in range(cnt.value):
                native.check(get(h, i, ctypes.byref(hv), ctypes.byref(pg)), "ls_neighbours_get")
                out.append((hv.value, pg.value.decode()))
            return out, dict(zip(("replayed", "accepted", "rejected", "deferred"), list(st)))
        finally:
            self._L.ls_neighbours_destroy(h)

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

            def __reduce__(self):  # picklable (reports cross GpuTaskPool's process boundary)
                return (_lazy_from_text, (self._ls_text, getattr(self, "_ls_hash", None)))

            def __eq__(self, other):  # equal to the reference object it stands for
                if isinstance(other, ir.TensorProgram):
                    return (self.buffers, self.root) == (other.buffers, other.root)
                return NotImplemented

            def __hash__(self):
                return hash((self.buffers, self.root))

        _LAZY = LazyProgram
    return _LAZY


def _lazy_from_text(text: str, h=None):
    p = lazy_program_class()(text)
    if h is not None:
        object.__setattr__(p, "_ls_hash", h)
    return p


def serialize_trace(t) -> str:
    """The reference's ``serialize_trace`` (`src/trace.py:82-88`), byte for
    byte, with each instruction's JSON line cached on the (frozen, never
    mutated) ``Instruction`` object: a mutated trace shares all but one
    instruction with its parent (`src/trace.py:287-310` builds the changed
    one with ``dataclasses.replace``), so re-serializing it costs one
    ``json.dumps`` instead of one per instruction."""
    lines = []
    if t.workload_hash is not None:
        lines.append(json.dumps({"workload_hash": t.workload_hash}, sort_keys=True))
    for ins in t.instructions:
        line = ins.__dict__.get("_ls_line")
        if line is None:
            line = json.dumps(ins.to_json(), sort_keys=True)
            object.__setattr__(ins, "_ls_line", line)
        lines.append(line)
    return "\n".join(lines) + ("\n" if lines else "")


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
            new_ins = tr.Instruction(d["op"], tuple(d.get("inputs", [])), d.get("attrs", {}),
                                     tuple(d.get("outputs", [])), d.get("decision"))
            object.__setattr__(new_ins, "_ls_line", line)  # the native line is its serialization
            ins.append(new_ins)
    return tr.Trace(tuple(ins), workload_hash=t.workload_hash, validated=True)


_NATIVE_VALIDATOR = None
_LAZY_CAND = None


def _lazy_candidate_class():
    """The reference's ``Candidate`` (`src/search.py:63-69`) whose ``features``
    and ``predicted`` are materialized on first access by the owning
    validator's batched featurization (the look-ahead)."""
    global _LAZY_CAND
    if _LAZY_CAND is None:
        S = loopsched().search

        class LazyCandidate(S.Candidate):
            def __init__(self, trace, program, h, owner, model, text):  # noqa: D107
                self.trace = trace
                self.program = program
                self.program_hash = h
                self._owner, self._model, self._text = owner, model, text
                self._f = self._p = None

            @property
            def features(self):
                if self._f is None:
                    self._owner._flush_lazy()
                return self._f

            @property
            def predicted(self):
                if self._f is None:
                    self._owner._flush_lazy()
                return self._p

        _LAZY_CAND = LazyCandidate
    return _LAZY_CAND


def native_validator_class():
    """``_Validator`` (`src/search.py:100-146`) with ``candidate`` replayed natively."""
    global _NATIVE_VALIDATOR
    if _NATIVE_VALIDATOR is None:
        ls = loopsched()
        S = ls.search
        base = S._Validator._ls_base if getattr(S._Validator, "_ls_dispatch", False) else S._Validator

        class NativeValidator(base):
            """``lookahead``: before a generation mutates its members, the
            single-decision neighbourhood of every member not expanded yet
            is replayed natively in one batch and the programs of its new
            structural hashes are featurized in one K7 launch (SURVEY.md
            §8f-2).  ``evolve``'s sequential proposals then find their
            features by hash (``features_by_hash``, the reference's own memo)
            instead of launching K7 one program at a time.  Only that memo
            is filled: the rng stream, the proposals, the verdicts and every
            decision of ``evolve`` are the reference's."""

            def __init__(self, e0, machine_spec=None, lookahead=False, featurize_batch=None):
                if machine_spec is None:
                    super().__init__(e0, ls.MachineSpec())
                else:
                    super().__init__(e0, machine_spec)
                self._rp = NativeReplayer(ls.ir.serialize(e0))
                self._lazy = lazy_program_class()
                self.native_calls = 0
                self.deferred = 0
                self.lookahead = lookahead
                self._featurize_batch = featurize_batch
                self._pending = []     # member traces not expanded yet
                self._expanded = set()
                self._building = False
                self._last = None
                self._lazies = []
                self._keys = {}          # id(trace) -> (trace, serialize_trace(trace)) of space traces
                self._orig_replay = ls.trace.replay
                self.expansions = 0
                self.neighbours = 0       # replayed by the look-ahead
                self.prefetched = 0       # programs featurized ahead

            # -- hooks driven by plugin.installed(lookahead=True) --
            def begin_evolve(self):
                self._building = True   # candidates returned until the first mutate are members

            def accepted(self):
                if self._last is not None:  # mh_accept kept the proposal just returned
                    self._pending.append(self._last.trace)

            def before_mutate(self, t):
                self._building = False
                k = getattr(t, "_ls_key", None) or serialize_trace(t)
                if k in self._expanded:
                    return
                keys = []
                for m in self._pending + [t]:
                    mk = getattr(m, "_ls_key", None) or serialize_trace(m)
                    if mk not in self._expanded:
                        self._expanded.add(mk)
                        keys.append(mk)
                self._pending = []
                self._expand(keys)

            def _expand(self, keys):
                new, stats = self._rp.neighbours(keys)
                self.expansions += 1
                self.neighbours += stats["replayed"]
                new = [(h, p) for h, p in new if h not in self.features_by_hash]
                self.prefetched += len(new)
                if not new:
                    return
                if self._featurize_batch is not None:
                    feats = self._featurize_batch([p for _, p in new], self.machine_spec)
                else:
                    feats = [S.featurize(self._lazy(p), self.machine_spec) for _, p in new]
                for (h, _), f in zip(new, feats):
                    self.features_by_hash[h] = f

            def _note(self, cand):
                self._last = cand
                if cand is not None and self._building:
                    self._pending.append(cand.trace)
                return cand

            def candidate(self, t, model):
                key = serialize_trace(t)
                if key in self.cache:
                    return self._note(self._revive(self.cache[key], model))
                (st, _idx, h, prog, norm, _reason), = self._rp.validate([key])
                self.native_calls += 1
                if st == REJECTED:
                    self.cache[key] = None
                    return self._note(None)
                if st == DEFER:
                    self.deferred += 1
                    return self._note(base.candidate(self, t, model))
                return self._note(self._store_native(key, self._trace(key, norm, t), self._lazy(prog), h, model))

            def resample(self, t, seed):
                """``replay(e0, t, "resample", seed)`` (`src/trace.py:163-198`)
                natively: the fresh candidates of `_fresh_candidate`
                (`src/search.py:149-159`)."""
                key = self._keys.get(id(t))
                if key is None or key[0] is not t:
                    key = (t, serialize_trace(t))
                    self._keys[id(t)] = key
                st, idx, h, prog, norm, reason = self._rp.resample(key[1], seed)
                self.native_calls += 1
                if st == REJECTED:
                    raise ls.trace.ReplayError(idx, reason)
                if st == DEFER:
                    self.deferred += 1
                    return self._orig_replay(self.e0, t, mode="resample", seed=seed)
                program = self._lazy(prog)
                object.__setattr__(program, "_ls_hash", h)
                return program, self._trace(key[1], norm, t)

            def from_replay(self, t, program, model):
                # a fresh (resampled) candidate: with the look-ahead its
                # features are computed lazily, all pending ones in one K7
                # batch on first use (evolve reads no feature or prediction
                # until the population is complete)
                native_h = getattr(program, "_ls_hash", None)
                if not self.lookahead and native_h is None:
                    return self._note(base.from_replay(self, t, program, model))
                key = getattr(t, "_ls_key", None) or serialize_trace(t)
                cand = self.cache.get(key)
                if cand is not None:
                    return self._note(self._revive(cand, model))
                text = getattr(program, "_ls_text", None) or ls.ir.serialize(program)
                h = native_h if native_h is not None else program_hash(text)
                if not self.lookahead:
                    return self._note(self._store_native(key, t, program, h, model))
                if h in self.features_by_hash:
                    return self._note(self._store_native(key, t, program, h, model))
                lazy = _lazy_candidate_class()(t, program, h, self, model, text)
                self._lazies.append(lazy)
                self.cache[key] = lazy
                return self._note(lazy)

            def _flush_lazy(self):
                todo = [c for c in self._lazies if c._f is None]
                self._lazies = []
                texts = {}
                for c in todo:
                    if c.program_hash not in self.features_by_hash:
                        texts.setdefault(c.program_hash, c._text)
                if texts:
                    hs = list(texts)
                    if self._featurize_batch is not None:
                        feats = self._featurize_batch([texts[h] for h in hs], self.machine_spec)
                    else:
                        feats = [S.featurize(self._lazy(texts[h]), self.machine_spec) for h in hs]
                    for h, f in zip(hs, feats):
                        self.features_by_hash[h] = f
                    self.prefetched += len(hs)
                for c in todo:
                    c._f = self.features_by_hash[c.program_hash]
                    c._p = self._predict(c.program, c._f, c._model)

            @staticmethod
            def _trace(key, norm, t):
                tr = normalized_trace(key, norm, t)
                object.__setattr__(tr, "_ls_key", norm)  # serialize_trace(tr), for the look-ahead
                return tr

            def prevalidate(self, traces):
                """Validate a batch of traces in one native call and store the
                accepted/rejected verdicts, so the sequential ``candidate``
                calls that follow are cache hits (featurize stays per program)."""
                keys, seen = [], set()
                for t in traces:
                    k = serialize_trace(t)
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
