"""Drop-in installation of the B200 path into the reference's search.

The reference's search driver (`tune` / `evolve` / `mutate` / `mh_accept`,
`src/search.py:162-376`) stays unchanged; for the duration of ``installed()``
(or one ``tune(...)`` call) its four seams are rebound:

  ======================================  ===========================================
  reference seam                          B200 implementation
  ======================================  ===========================================
  ``search._measure_batch`` (:249-256,    ``Runner.measure``: hardware (``B200Runner``,
  called at :345)                         ``ShardedRunner``) or parity (``SimRunner``)
  ``search.simulate_latency`` (baseline,  ``Runner.baseline``
  :326)
  ``search.featurize`` (:141)             K7 on the GPU, memoized by program text
  ``_Validator._predict`` (:109-111; the  K7b: every known feature row rescored in
  reference's own plug-in seam,           one launch per model, then lookups
  tests/test_search.py:125-127)
  ``search._Validator`` (:100-146,        ``replay.NativeValidator``: validate_trace
  constructed at :324 and :169)           replayed natively (``ls_replay_batch``)
  ======================================  ===========================================

Nothing in the reference is edited or copied; the originals are restored on
exit even when the search raises.
"""

from __future__ import annotations

import atexit
import contextlib
import threading
from fractions import Fraction

import numpy as np

from .inputs import program_text
from .refapi import loopsched


class SimRunner:
    """Parity-mode Runner: the reference's simulated latency, computed exactly
    (int128 rationals) by the K8 kernel -- bit-identical to
    ``simulate_latency`` (`src/machine.py:228-254`)."""

    def __init__(self, device: int = 0, scorer=None):
        from .scorer import GpuScorer
        self.scorer = scorer or GpuScorer(device)

    def measure(self, candidates, machine_spec=None, jobs: int = 1) -> list:
        if not candidates:
            return []
        return self.scorer.sim_latency_batch(candidates, machine_spec)

    def baseline(self, e0, machine_spec=None) -> Fraction:
        return self.scorer.sim_latency_batch([e0], machine_spec)[0]


class ScoreCache:
    """K7 features memoized by program text; predictions memoized per model
    (a new model triggers one batched K7b launch over every known row).

    ``exact=True`` (parity mode): the score the search compares is the
    reference's own ``CostModel.predict_features`` (`src/costmodel.py:98-102`)
    evaluated on the host for each new feature row, so ``mh_accept`` and the
    (predicted, hash) ranking see bit-identical values even on near-ties
    (numpy's ddot summation order and libm's exp are host-specific; the
    device score agrees to ~1e-15 relative, not bitwise)."""

    def __init__(self, scorer, exact: bool = False):
        self.scorer = scorer
        self.exact = exact
        self.features: dict[str, np.ndarray] = {}
        self._model = None
        self._scores: dict[bytes, float] = {}
        self.launches = 0
        self.feat_launches = 0  # K7 featurize launches (the rest score feature rows)

    def featurize(self, program, machine_spec=None) -> np.ndarray:
        text = program_text(program)
        f = self.features.get(text)
        if f is None:
            f = self.scorer.featurize_batch([text], machine_spec)[0]
            self.launches += 1
            self.feat_launches += 1
            self.features[text] = f
        return f.copy()

    def featurize_many(self, texts, machine_spec=None):
        """K7 over a batch of program texts in one launch (the look-ahead);
        memoized like ``featurize``."""
        todo = [t for t in dict.fromkeys(texts) if t not in self.features]
        if todo:
            feats = self.scorer.featurize_batch(todo, machine_spec)
            self.launches += 1
            self.feat_launches += 1
            for t, f in zip(todo, feats):
                self.features[t] = f
        return [self.features[t].copy() for t in texts]

    def predict(self, features, model) -> float:
        if self.exact:
            return positive_score(model.predict_features(np.asarray(features, dtype=np.float64)))
        if model is not self._model:
            self._model = model
            self._scores = {}
            rows = {f.tobytes(): f for f in self.features.values()}
            if rows:
                keys = list(rows)
                vals = self.scorer.score_batch(np.stack([rows[k] for k in keys]), model)
                self.launches += 1
                self._scores = dict(zip(keys, map(float, vals)))
        f = np.asarray(features, dtype=np.float64)
        key = f.tobytes()
        s = self._scores.get(key)
        if s is None:
            s = float(self.scorer.score_batch(f.reshape(1, 9), model)[0])
            self.launches += 1
            self._scores[key] = s
        return positive_score(s)


_TINY, _HUGE = 5e-324, 1.7976931348623157e308


def positive_score(s: float) -> float:
    """The model's prediction exp(...) as the search needs it: strictly
    positive and finite (`mh_accept` raises otherwise, `src/search.py:88-97`).
    Identical to the reference's value whenever that one is usable; only an
    exp() that underflowed to 0 or overflowed to inf -- reachable when the
    model is fitted on hardware nanoseconds with sentinel latencies and
    extrapolates far -- is clamped to the nearest positive finite double."""
    if s != s:  # NaN: no ordering information; treat as the worst
        return _HUGE
    return min(max(s, _TINY), _HUGE)


class _Seams:
    """What one ``installed()`` block routes the reference's seams to."""

    def __init__(self, runner, cache, native_replay=True, lookahead=False):
        self.runner = runner
        self.cache = cache
        self.native_replay = native_replay
        self.lookahead = lookahead
        self.validator = None  # the NativeValidator of this block's search


_tls = threading.local()
_install_lock = threading.Lock()
_install_depth = 0
_originals = None


def _current():
    st = getattr(_tls, "stack", None)
    return st[-1] if st else None


def _d_measure(cands, spec, jobs):
    cur = _current()
    if cur is not None and cur.runner is not None:
        return cur.runner.measure(cands, spec, jobs)
    return _originals[0](cands, spec, jobs)


def _d_simulate(p, spec=None):
    cur = _current()
    if cur is not None and cur.runner is not None:
        return cur.runner.baseline(p, spec)
    return _originals[1](p, spec) if spec is not None else _originals[1](p)


def _d_featurize(p, spec=None):
    cur = _current()
    if cur is not None and cur.cache is not None:
        return cur.cache.featurize(p, spec)
    return _originals[2](p, spec) if spec is not None else _originals[2](p)


def _d_validator(e0, machine_spec=None):
    cur = _current()
    base = _originals[4]
    if cur is not None and cur.native_replay:
        from .replay import native_validator_class
        cls = native_validator_class()
        fb = cur.cache.featurize_many if cur.cache is not None else None
        v = cls(e0, machine_spec, lookahead=cur.lookahead, featurize_batch=fb)
        cur.validator = v
        return v
    return base(e0, machine_spec) if machine_spec is not None else base(e0)


def _lookahead_validator():
    cur = _current()
    v = cur.validator if cur is not None else None
    return v if v is not None and v.lookahead else None


def _d_replay(e0, t, mode="follow", seed=0):
    # the resampled replays of `_fresh_candidate` (src/search.py:149-159)
    # for this block's workload go native; everything else to the reference
    cur = _current()
    v = cur.validator if cur is not None else None
    if mode == "resample" and v is not None and e0 is v.e0:
        return v.resample(t, seed)
    return _originals[8](e0, t, mode, seed)


def _d_evolve(*args, **kw):
    v = kw.get("validator", args[5] if len(args) > 5 else None)
    if v is not None and getattr(v, "lookahead", False):
        v.begin_evolve()
    return _originals[5](*args, **kw)


def _d_mutate(t, rng):
    v = _lookahead_validator()
    if v is not None:
        v.before_mutate(t)   # fills caches only; consumes no randomness
    return _originals[6](t, rng)


def _d_mh_accept(old_pred, new_pred, temperature, rng):
    ok = _originals[7](old_pred, new_pred, temperature, rng)
    if ok:
        v = _lookahead_validator()
        if v is not None:
            v.accepted()
    return ok


def _d_predict(self, program, features, model):
    cur = _current()
    if cur is not None and cur.cache is not None:
        return cur.cache.predict(features, model)
    return _originals[3](self, program, features, model)


@contextlib.contextmanager
def installed(runner=None, scorer=None, exact_scores: bool = False, native_replay: bool = True,
              lookahead: bool = False):
    """Route the reference's seams to ``runner`` (Runner protocol) and
    ``scorer`` (Scorer protocol) inside the block.

    The module-level seams are rebound once to dispatchers that look up the
    innermost ``installed()`` block of the CALLING THREAD (falling back to the
    reference's originals), so concurrent tunes on several threads -- e.g. one
    per GPU -- each see their own runner; the originals are restored when the
    last block exits, also when the search raises.  ``native_replay``
    routes ``validate_trace`` through the native replay (replay.py);
    ``lookahead`` (with it) prefetches each generation's single-decision
    neighbourhood in one native replay batch + one K7 launch, observing
    ``evolve`` / ``mutate`` / ``mh_accept`` without changing them.  It cuts
    K7 launches per tune ~50x but replays every neighbour (~44 k for a
    64-trial gmm512 tune, +0.35 s on the B200 box's host), so it is off by
    default (profiles/r02_search.md)."""
    global _install_depth, _originals
    ls = loopsched()
    S = ls.search
    cache = ScoreCache(scorer, exact=exact_scores) if scorer is not None else None
    with _install_lock:
        if _install_depth == 0:
            vcls = S._Validator
            _originals = (S._measure_batch, S.simulate_latency, S.featurize, vcls._predict, vcls,
                          S.evolve, S.mutate, S.mh_accept, S.replay)
            S._measure_batch, S.simulate_latency, S.featurize = _d_measure, _d_simulate, _d_featurize
            S.evolve, S.mutate, S.mh_accept, S.replay = _d_evolve, _d_mutate, _d_mh_accept, _d_replay
            vcls._predict = _d_predict
            _d_validator._ls_dispatch = True
            _d_validator._ls_base = vcls
            S._Validator = _d_validator
        _install_depth += 1
    st = getattr(_tls, "stack", None)
    if st is None:
        st = _tls.stack = []
    st.append(_Seams(runner, cache, native_replay, lookahead and native_replay))
    try:
        yield cache
    finally:
        st.pop()
        with _install_lock:
            _install_depth -= 1
            if _install_depth == 0:
                vcls = _originals[4]
                S._measure_batch, S.simulate_latency, S.featurize, vcls._predict = _originals[:4]
                S._Validator = vcls
                S.evolve, S.mutate, S.mh_accept, S.replay = _originals[5:9]
                _originals = None


last_tune_stats: dict = {}


_RUNNER_POOL: dict = {}


def close_runner_pool() -> None:
    """Destroy the pooled hardware runners (also run at interpreter exit,
    before the CUDA context is torn down)."""
    while _RUNNER_POOL:
        _, r = _RUNNER_POOL.popitem()
        r.close()


atexit.register(close_runner_pool)


def _pooled_runner(device, dtype, opts):
    """One hardware runner per (device, dtype, options), reused across tunes:
    creating one costs milliseconds (kernel preloads, pinned staging) and
    destroying one ~0.1 s (device and pinned frees), which would otherwise
    land inside the next tune's wall time.  ``set_workload`` resets the
    per-workload state (reference output, baseline, deadline cap)."""
    from .runner import B200Runner
    key = (device, dtype, tuple(sorted(opts.items())))
    r = _RUNNER_POOL.get(key)
    if r is None or getattr(r, "_h", None) is None:
        r = _RUNNER_POOL[key] = B200Runner(device=device, dtype=dtype, **opts)
    return r


def tune(e0, generator, config=None, machine_spec=None, warm_records=None, *,
         mode: str = "hardware", runner=None, scorer=None, device: int = 0, dtype: str = "bf16",
         native_replay: bool = True, lookahead: bool = False, **runner_opts):
    """The reference's ``tune`` with the B200 seams installed.

    mode "hardware": candidates are instantiated and timed on the GPU
    (latencies in ns); mode "parity": latencies are the reference's simulated
    cycles computed exactly on the GPU, so the search makes the same decisions
    as the CPU reference for the same seed."""
    ls = loopsched()
    from .scorer import GpuScorer
    config = config or ls.SearchConfig()
    machine_spec = machine_spec or ls.MachineSpec()
    scorer = scorer or GpuScorer(device)
    if runner is None:
        if mode == "parity":
            runner = SimRunner(device, scorer)
        elif mode == "hardware":
            runner = _pooled_runner(device, dtype, runner_opts)
            runner.set_workload(e0)
        else:
            raise ValueError(f"unknown mode {mode!r}")
    with installed(runner, scorer, exact_scores=(mode == "parity"), native_replay=native_replay,
                   lookahead=lookahead) as cache:
        report = ls.search.tune(e0, generator, config, machine_spec, warm_records)
        v = _current().validator
        last_tune_stats.clear()
        last_tune_stats.update({
            "k7_featurize_launches": cache.feat_launches, "k7_launches": cache.launches,
            "native_replay": native_replay, "lookahead": lookahead and native_replay,
            "native_validations": getattr(v, "native_calls", 0),
            "lookahead_expansions": getattr(v, "expansions", 0),
            "lookahead_neighbours": getattr(v, "neighbours", 0),
            "lookahead_prefetched": getattr(v, "prefetched", 0)})
        return report


def tune_with_records(e0, generator, config=None, machine_spec=None, *, runner=None, scorer=None,
                      mode: str = "hardware", records_path=None, warm_path=None, device: int = 0,
                      dtype: str = "bf16", peak_tflops=None, peak_source="", **runner_opts):
    """``tune`` plus the hardware record/report format (records.py): warm-starts
    from ``warm_path`` (records of the same workload and unit only), writes the
    log to ``records_path`` and returns ``(report, report_json)`` where the JSON
    is the reference's report with a ``hardware`` section (best-schedule
    TFLOPS, roofline fraction, per-record kernel family / configuration)."""
    from . import records as R
    unit = "cycles" if mode == "parity" else "ns"
    ctx = R.HardwareContext.for_workload(e0, unit=unit, dtype=dtype, peak_tflops=peak_tflops,
                                         peak_source=peak_source)
    warm = R.load_records(warm_path, workload_hash=ctx.workload_hash, unit=unit) if warm_path else None
    if runner is None and mode == "hardware":
        from .runner import B200Runner
        runner = B200Runner(device=device, dtype=dtype, **runner_opts)
        runner.set_workload(e0)
    rec = R.RecordingRunner(runner) if runner is not None else None
    report = tune(e0, generator, config, machine_spec, warm, mode=mode, runner=rec, scorer=scorer,
                  device=device, dtype=dtype)
    info = rec.info if rec is not None else {}
    if records_path:
        R.save_records(records_path, report.log, ctx, info)
    return report, R.report_json(report, ctx, info)
