"""Whole-network tuning: task extraction + trial allocation (SURVEY.md §8f-3,
BASELINE config 5 "BERT-base end-to-end: all extracted tasks tuned, 2000
trials over 8xB200").

The reference tunes one workload per ``tune`` call and has no multi-task
scheduler (`SPEC.md:656`).  ``TaskScheduler`` drives the reference's
unchanged ``tune`` (through ``plugin.tune``, so candidates are measured by the
B200 Runner -- one GPU or ``ShardedRunner`` over all GPUs of the box) in
rounds of ``round_trials`` per task, carrying each task's measured records
forward as ``warm_records`` (`src/search.py:328-329`) so every round refits
the cost model on everything measured for that task so far.

Allocation is the gradient rule of Ansor's task scheduler (Zheng et al.,
OSDI'20, §6): after one warm-up round per task, the next round goes to the
task with the largest estimated decrease of the network objective
``f = sum_i w_i * best_i`` (``w_i`` = occurrences of the operator in the
network) per trial:

    g_i = w_i * ( alpha * (best_i(t_i - dt_i) - best_i(t_i)) / dt_i
                  + (1 - alpha) * best_i(t_i) / t_i )

the first term is the recent improvement rate, the second an optimistic
estimate that keeps under-explored tasks in play.  Exhausted tasks (the
reference's ``report.exhausted``) leave the pool.  Everything is
deterministic per ``seed``.

Repeat schedules: each round is a fresh reference ``tune`` whose
``state.measured`` starts empty, so it can propose programs an earlier round
already measured.  ``CachingRunner`` answers those from the task's records
(by ``program_hash``) without touching the GPU, only newly measured programs
count toward the budget, and the warm-start records are de-duplicated by
hash so the refit does not over-weight repeats.

Task parallelism (``run(parallel=G)``): synchronous waves -- the G tasks with
the largest gradients (distinct tasks, deterministic tie-break) each run one
round at the same time, one per GPU (``GpuTaskPool``: a worker process per
device running the reference ``tune`` with the B200 seams), and the
allocation state is updated in task order once the wave completes.  The
allocation therefore depends only on the round results, never on which
worker finished first.
"""

from __future__ import annotations

import hashlib
import os
from dataclasses import dataclass, field
from fractions import Fraction
from typing import Callable, Optional

from .refapi import loopsched


@dataclass
class Task:
    name: str
    e0: object                  # reference TensorProgram
    weight: int                 # occurrences in the network
    trials: int = 0
    rounds: int = 0
    baseline: Optional[Fraction] = None
    best: Optional[Fraction] = None
    history: list = field(default_factory=list)   # (trials, best) after each round
    records: list = field(default_factory=list)   # reference TuningRecords
    exhausted: bool = False
    best_trace: Optional[object] = None


def bert_tasks(seq: int = 128, layers: int = 12, scale: int = 1):
    """BERT-base operator tasks with their network weight (per-layer count x
    layers).  ``scale`` divides every dimension (for quick CPU tests)."""
    from .workloads import bert_base_tasks, batch_matmul
    ls = loopsched()
    if scale == 1:
        return [Task(name, e0, count * layers) for name, e0, count in bert_base_tasks(seq)]
    s, h, f, d = seq // scale, 768 // scale, 3072 // scale, 64 // scale
    heads = max(1, 12 // scale)
    return [Task("dense_qkvo", ls.gmm(s, h, h), 4 * layers),
            Task("ffn_in", ls.gmm(s, f, h), layers),
            Task("ffn_out", ls.gmm(s, h, f), layers),
            Task("attn_qk", batch_matmul(heads, s, s, d), layers),
            Task("attn_pv", batch_matmul(heads, s, d, s), layers)]


class CachingRunner:
    """Runner protocol over ``base``: candidates whose ``program_hash`` is
    already in ``known`` (hash -> latency, from earlier rounds of the task)
    are answered from it; only the rest reach the device.  ``fresh`` counts
    the newly measured programs."""

    def __init__(self, base, known=None):
        self.base = base
        self.known = dict(known or {})
        self.fresh = 0

    def measure(self, candidates, machine_spec=None, jobs: int = 1) -> list:
        todo = [c for c in candidates if c.program_hash not in self.known]
        if todo:
            lats = self.base.measure(todo, machine_spec, jobs)
            for c, lat in zip(todo, lats):
                self.known[c.program_hash] = lat
            self.fresh += len(todo)
        return [self.known[c.program_hash] for c in candidates]

    def baseline(self, e0, machine_spec=None):
        return self.base.baseline(e0, machine_spec)


class _CountingSimRunner:
    """Reference Runner (``simulate_latency``) behind the CachingRunner when no
    device runner is given (CPU tests / parity mode)."""

    def measure(self, candidates, machine_spec=None, jobs: int = 1):
        ls = loopsched()
        return [ls.simulate_latency(c.program, machine_spec or ls.MachineSpec()) for c in candidates]

    def baseline(self, e0, machine_spec=None):
        ls = loopsched()
        return ls.simulate_latency(e0, machine_spec or ls.MachineSpec())


def dedup_records(records):
    """First record per program hash, in order."""
    seen, out = set(), []
    for r in records:
        if r.program_hash in seen:
            continue
        seen.add(r.program_hash)
        out.append(r)
    return out


class TaskScheduler:
    def __init__(self, tasks, total_trials: int, *, round_trials: int = 64, batch: int = 16,
                 population: int = 64, seed: int = 0, alpha: float = 0.2,
                 generator_for: Optional[Callable] = None,
                 runner_for: Optional[Callable] = None, scorer=None, mode: str = "hardware",
                 tune_fn: Optional[Callable] = None):
        self.tasks = list(tasks)
        self.total = int(total_trials)
        self.round_trials = int(round_trials)
        self.batch, self.population = batch, population
        self.seed, self.alpha = seed, alpha
        ls = loopsched()
        self.generator_for = generator_for or (lambda task: ls.default_space())
        self.runner_for = runner_for or (lambda task: None)
        self.scorer = scorer
        self.mode = mode
        self.tune_fn = tune_fn
        self.spent = 0
        self.log: list = []   # (round index, task name, new trials, best)

    # -- objective / gradient ------------------------------------------------
    def objective(self) -> Optional[Fraction]:
        if any(t.best is None for t in self.tasks):
            return None
        return sum((Fraction(t.weight) * t.best for t in self.tasks), Fraction(0))

    def gradient(self, t: Task) -> float:
        if t.best is None or t.trials == 0:
            return float("inf")
        if len(t.history) >= 2:
            (t0, b0), (t1, b1) = t.history[-2], t.history[-1]
            recent = float(b0 - b1) / max(1, t1 - t0)
        else:
            recent = float(t.baseline - t.best) / max(1, t.trials) if t.baseline is not None else 0.0
        optimistic = float(t.best) / t.trials
        return t.weight * (self.alpha * recent + (1.0 - self.alpha) * optimistic)

    # -- one round of one task ------------------------------------------------
    def _round_seed(self, t: Task) -> int:
        h = hashlib.sha256(f"{self.seed}/{t.name}/{t.rounds}".encode()).digest()
        return int.from_bytes(h[:6], "little")

    def round_config(self, t: Task, want: int):
        ls = loopsched()
        return ls.SearchConfig(trials=want, batch=min(self.batch, want), population=self.population,
                               seed=self._round_seed(t))

    def execute_round(self, t: Task, cfg):
        """Run one reference ``tune`` round of ``t`` here; returns (report,
        newly measured programs)."""
        known = {r.program_hash: r.latency for r in t.records}
        warm = t.records or None
        base = self.runner_for(t)
        if self.tune_fn is not None:
            from . import plugin
            cache = CachingRunner(base if base is not None else _CountingSimRunner(), known)
            with plugin.installed(runner=cache):   # per-thread seams: waves may run on threads
                report = self.tune_fn(t.e0, self.generator_for(t), cfg, warm)
            return report, cache.fresh
        from . import plugin
        if base is None:
            return plugin.tune(t.e0, self.generator_for(t), cfg, None, warm, mode=self.mode,
                               scorer=self.scorer), None
        cache = CachingRunner(base, known)
        report = plugin.tune(t.e0, self.generator_for(t), cfg, None, warm, mode=self.mode, runner=cache,
                             scorer=self.scorer)
        return report, cache.fresh

    def apply_round(self, t: Task, report, fresh) -> None:
        """Fold one round's report into the task and the allocation state."""
        n = len(report.log) if fresh is None else fresh
        t.rounds += 1
        t.trials += n
        self.spent += n
        t.records = dedup_records(list(t.records) + list(report.log))
        if t.baseline is None:
            t.baseline = report.baseline_latency
        if report.best is not None and (t.best is None or report.best.latency < t.best):
            t.best = report.best.latency
            t.best_trace = report.best.trace
        if t.best is None:
            t.best = t.baseline
        t.history.append((t.trials, t.best))
        if report.exhausted or n == 0:
            t.exhausted = True
        self.log.append((len(self.log), t.name, n, t.best))

    def tune_round(self, t: Task) -> None:
        want = min(self.round_trials, self.total - self.spent)
        if want <= 0:
            return
        report, fresh = self.execute_round(t, self.round_config(t, want))
        self.apply_round(t, report, fresh)

    # -- the allocation loop --------------------------------------------------
    def _pick(self, k: int):
        pool = [t for t in self.tasks if not t.exhausted]
        ranked = sorted(pool, key=lambda t: (-self.gradient(t), self.tasks.index(t)))
        return ranked[:k]

    def run(self, parallel: int = 1, submit: Optional[Callable] = None) -> dict:
        """Allocate the budget.  ``parallel`` > 1 runs waves of that many
        distinct tasks at once through ``submit(scheduler, task, cfg) ->
        future`` (``GpuTaskPool.submit``: one round per GPU; any executor
        whose futures return ``(report, fresh)`` works)."""
        if parallel <= 1 or submit is None:
            for t in self.tasks:                      # warm-up: one round each
                if self.spent >= self.total:
                    break
                self.tune_round(t)
            while self.spent < self.total:
                pool = self._pick(1)
                if not pool:
                    break
                best = pool[0]
                before = self.spent
                self.tune_round(best)
                if self.spent == before:
                    best.exhausted = True
            return self.summary()
        warm = list(self.tasks)
        while self.spent < self.total:
            if warm:
                wave, warm = warm[:parallel], warm[parallel:]
            else:
                wave = self._pick(parallel)
            if not wave:
                break
            left = self.total - self.spent
            jobs = []
            for t in wave:   # budget split over the wave in task order (deterministic)
                want = min(self.round_trials, left)
                if want <= 0:
                    break
                left -= want
                jobs.append((t, submit(self, t, self.round_config(t, want))))
            if not jobs:
                break
            for t, fut in jobs:            # fold in task order, not completion order
                report, fresh = fut.result()
                self.apply_round(t, report, fresh)   # a round with nothing new exhausts its task
        return self.summary()

    def summary(self) -> dict:
        obj = self.objective()
        base = sum((Fraction(t.weight) * t.baseline for t in self.tasks if t.baseline is not None), Fraction(0))
        return {
            "trials": self.spent, "budget": self.total,
            "objective": None if obj is None else float(obj),
            "objective_exact": None if obj is None else str(obj),
            "baseline_objective": float(base),
            "speedup": None if not obj else float(base / obj),
            "tasks": [{"name": t.name, "weight": t.weight, "trials": t.trials, "rounds": t.rounds,
                       "baseline": None if t.baseline is None else float(t.baseline),
                       "best": None if t.best is None else float(t.best),
                       "speedup": None if not t.best or t.baseline is None else float(t.baseline / t.best),
                       "exhausted": t.exhausted} for t in self.tasks],
            "allocation": [{"round": i, "task": name, "trials": n, "best": float(b)} for i, name, n, b in self.log],
        }


def _gpu_worker(conn, device: int, runner_opts: dict, space_doc):
    """One GPU: the reference ``tune`` with the B200 seams, one B200Runner per
    task (workload uploaded once), latencies cached by program hash."""
    os.environ["CUDA_VISIBLE_DEVICES"] = str(device)
    from . import plugin
    from .runner import B200Runner
    from .scorer import GpuScorer
    from .tensor_core import space_from_config
    ls = loopsched()
    scorer = GpuScorer(0)
    runners = {}
    try:
        while True:
            msg = conn.recv()
            if msg is None:
                break
            name, e0_text, cfg_kw, records, mode, dtype = msg
            try:
                e0 = ls.ir.deserialize(e0_text)
                cfg = ls.SearchConfig(**cfg_kw)
                base = None
                if mode == "hardware":
                    if name not in runners:
                        r = B200Runner(device=0, dtype=dtype, carry_best=True, **runner_opts)
                        r.set_workload(e0)
                        runners[name] = r
                    base = runners[name]
                    cache = CachingRunner(base, {r.program_hash: r.latency for r in records})
                    rep = plugin.tune(e0, space_from_config(space_doc), cfg, None, records or None,
                                      mode=mode, runner=cache, scorer=scorer)
                    conn.send(("ok", (rep, cache.fresh)))
                else:
                    rep = plugin.tune(e0, space_from_config(space_doc), cfg, None, records or None,
                                      mode=mode, scorer=scorer)
                    conn.send(("ok", (rep, None)))
            except Exception as exc:
                conn.send(("err", repr(exc)))
    finally:
        for r in runners.values():
            r.close()
        conn.close()


class GpuTaskPool:
    """One worker process per GPU for ``TaskScheduler.run(parallel=...)``.
    Each ``submit`` goes to a free worker; futures resolve to
    ``(report, newly measured)``."""

    def __init__(self, devices, space_doc: dict, dtype: str = "bf16", mode: str = "hardware", **runner_opts):
        import multiprocessing as mp
        from concurrent.futures import ThreadPoolExecutor
        ctx = mp.get_context("spawn")
        self.mode, self.dtype = mode, dtype
        self._conns, self._procs = [], []
        for d in devices:
            a, b = ctx.Pipe()
            p = ctx.Process(target=_gpu_worker, args=(b, d, runner_opts, space_doc), daemon=True)
            p.start()
            self._conns.append(a)
            self._procs.append(p)
        import queue
        self._free = queue.Queue()
        for c in self._conns:
            self._free.put(c)
        self._pool = ThreadPoolExecutor(max_workers=len(self._conns))

    def _run(self, name, e0_text, cfg_kw, records):
        conn = self._free.get()
        try:
            conn.send((name, e0_text, cfg_kw, records, self.mode, self.dtype))
            st, val = conn.recv()
        finally:
            self._free.put(conn)
        if st != "ok":
            raise RuntimeError(f"task round {name} failed: {val}")
        return val

    def submit(self, sched, t: Task, cfg):
        ls = loopsched()
        cfg_kw = {k: getattr(cfg, k) for k in cfg.__dataclass_fields__}
        return self._pool.submit(self._run, t.name, ls.ir.serialize(t.e0), cfg_kw, list(t.records))

    def close(self):
        for c in self._conns:
            try:
                c.send(None)
            except Exception:
                pass
        for p in self._procs:
            p.join(timeout=30)
        self._pool.shutdown()
        self._conns, self._procs = [], []
