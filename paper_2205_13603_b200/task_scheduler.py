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
"""

from __future__ import annotations

import hashlib
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
        self.log: list = []   # (round index, task name, trials, best)

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

    def tune_round(self, t: Task) -> None:
        ls = loopsched()
        want = min(self.round_trials, self.total - self.spent)
        if want <= 0:
            return
        cfg = ls.SearchConfig(trials=want, batch=min(self.batch, want), population=self.population,
                              seed=self._round_seed(t))
        if self.tune_fn is not None:
            report = self.tune_fn(t.e0, self.generator_for(t), cfg, t.records or None)
        else:
            from . import plugin
            report = plugin.tune(t.e0, self.generator_for(t), cfg, None, t.records or None, mode=self.mode,
                                 runner=self.runner_for(t), scorer=self.scorer)
        n = len(report.log)
        t.rounds += 1
        t.trials += n
        self.spent += n
        t.records = list(t.records) + list(report.log)
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

    # -- the allocation loop --------------------------------------------------
    def run(self) -> dict:
        for t in self.tasks:                      # warm-up: one round each
            if self.spent >= self.total:
                break
            self.tune_round(t)
        while self.spent < self.total:
            pool = [t for t in self.tasks if not t.exhausted]
            if not pool:
                break
            best = max(pool, key=lambda t: (self.gradient(t), -self.tasks.index(t)))
            before = self.spent
            self.tune_round(best)
            if self.spent == before:
                best.exhausted = True
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
