"""Hardware-latency tuning records and reports.

The reference keeps its search log in two formats:

* ``TuningReport.to_json`` (`src/search.py:280-312`): baseline, best, the log
  of every measured trace with ``float`` and exact ``str(Fraction)`` latency;
* ``save_records`` / ``load_records`` (`src/search.py:383-405`): JSON lines of
  ``{trace, latency (float), features, hash}`` that warm-start the cost model
  (``tune(..., warm_records=...)``, `src/search.py:328-329`).

Both assume one latency unit (simulated cycles).  On the B200 path a latency
is a measured duration in nanoseconds (``Fraction`` at picosecond
resolution, `runner.ns_fraction`), produced by a named device, dtype and
kernel family.  This module adds, without touching the reference:

* ``HardwareContext`` -- unit, device, dtype, peak and workload FLOPs;
* ``RecordingRunner`` -- wraps a Runner and keeps each measured program's
  kernel family / configuration / status by ``program_hash``;
* ``report_json`` -- the reference's report plus a ``hardware`` section:
  best-schedule TFLOPS and roofline fraction, per-record TFLOPS, family, cfg;
* ``save_records`` / ``load_records`` -- JSON lines that keep the exact
  latency (``str(Fraction)``), its unit and the workload hash, and load back
  into the reference's own ``TuningRecord`` (via its ``deserialize_trace``)
  for a warm start; records of another unit or workload are refused, since a
  model fitted on simulated cycles must not be mixed with nanoseconds.
"""

from __future__ import annotations

import json
from dataclasses import asdict, dataclass, field
from fractions import Fraction
from typing import Optional

import numpy as np

from .inputs import program_text
from .refapi import loopsched

RECORD_VERSION = 1


def contraction_flops(e0) -> float:
    """2 x the iteration count of every reduction statement of the
    unscheduled program (elementwise stages such as a pad are not counted)."""
    doc = json.loads(program_text(e0))

    def walk(stmts):
        tot = 0
        for st in stmts:
            if "loop" in st:
                tot += st["loop"]["extent"] * walk(st["loop"]["body"])
            elif "compute" in st and "init" in st["compute"]:
                tot += 1
        return tot

    return 2.0 * walk(doc["root"])


@dataclass
class HardwareContext:
    unit: str = "ns"                 # "ns" (hardware runner) or "cycles" (simulated, parity mode)
    device: str = "B200"
    dtype: str = "bf16"
    workload_hash: int = 0
    flops: float = 0.0               # per candidate execution
    peak_tflops: Optional[float] = None
    peak_source: str = ""
    extra: dict = field(default_factory=dict)

    @classmethod
    def for_workload(cls, e0, unit="ns", device="B200", dtype="bf16", peak_tflops=None, peak_source=""):
        ls = loopsched()
        prog = ls.ir.deserialize(e0) if isinstance(e0, str) else e0
        return cls(unit=unit, device=device, dtype=dtype, workload_hash=ls.ir.structural_hash(prog),
                   flops=contraction_flops(e0), peak_tflops=peak_tflops, peak_source=peak_source)

    def tflops(self, latency: Fraction) -> Optional[float]:
        if self.unit != "ns" or not latency or not self.flops:
            return None
        return self.flops / (float(latency) * 1e-9) / 1e12


class RecordingRunner:
    """Runner protocol wrapper: forwards to ``runner`` and keeps the per-program
    hardware outcome (``runner.last_results``) by the candidate's program hash."""

    def __init__(self, runner):
        self.runner = runner
        self.info: dict[int, dict] = {}

    def measure(self, candidates, machine_spec=None, jobs: int = 1) -> list:
        lat = self.runner.measure(candidates, machine_spec, jobs)
        results = getattr(self.runner, "last_results", None) or []
        for c, r in zip(candidates, results):
            self.info[c.program_hash] = {k: r[k] for k in ("family", "cfg", "status", "repeats") if k in r}
        return lat

    def baseline(self, e0, machine_spec=None):
        return self.runner.baseline(e0, machine_spec)


def report_json(report, ctx: HardwareContext, info: Optional[dict] = None, timestamp: bool = False) -> dict:
    """``report.to_json`` (unchanged keys) + a ``hardware`` section."""
    doc = report.to_json(timestamp=timestamp)
    info = info or {}
    per = []
    for rec in report.log:
        row = {"hash": rec.program_hash, "tflops": ctx.tflops(rec.latency)}
        row.update(info.get(rec.program_hash, {}))
        per.append(row)
    hw = {"version": RECORD_VERSION, "context": asdict(ctx), "records": per,
          "baseline_tflops": ctx.tflops(report.baseline_latency)}
    if report.best is not None:
        t = ctx.tflops(report.best.latency)
        hw["best"] = {"tflops": t, "latency_unit": ctx.unit, **info.get(report.best.program_hash, {})}
        if t is not None and ctx.peak_tflops:
            fam = hw["best"].get("family")
            bound = ("fp32-simt" if fam not in (None, "tcgen05", "tcgen05_conv") and ctx.dtype != "bf16"
                     else "tensor")
            hw["best"]["roofline"] = {"bound": bound, "peak": ctx.peak_tflops, "unit": "TFLOP/s",
                                      "frac": t / ctx.peak_tflops, "peak_source": ctx.peak_source}
    doc["hardware"] = hw
    return doc


def save_records(path: str, records, ctx: HardwareContext, info: Optional[dict] = None) -> None:
    """JSON lines; the exact latency survives the round trip."""
    info = info or {}
    with open(path, "w") as fh:
        for r in records:
            row = {"version": RECORD_VERSION, "workload": ctx.workload_hash, "unit": ctx.unit,
                   "device": ctx.device, "dtype": ctx.dtype,
                   "trace": [i.to_json() for i in r.trace.instructions],
                   "latency": float(r.latency), "latency_exact": str(Fraction(r.latency)),
                   "features": list(map(float, r.features)), "hash": r.program_hash,
                   "tflops": ctx.tflops(r.latency)}
            row.update({k: v for k, v in info.get(r.program_hash, {}).items() if k not in row})
            fh.write(json.dumps(row, sort_keys=True) + "\n")


def load_records(path: str, *, workload_hash: Optional[int] = None, unit: Optional[str] = None) -> list:
    """Reference ``TuningRecord`` objects for ``tune(..., warm_records=...)``.
    Raises ``ValueError`` on a unit or workload mismatch."""
    ls = loopsched()
    out = []
    with open(path) as fh:
        for n, line in enumerate(fh, 1):
            if not line.strip():
                continue
            doc = json.loads(line)
            if unit is not None and doc.get("unit", "cycles") != unit:
                raise ValueError(f"{path}:{n}: record unit {doc.get('unit', 'cycles')!r}, expected {unit!r}")
            if workload_hash is not None and doc.get("workload") not in (None, workload_hash):
                raise ValueError(f"{path}:{n}: record of workload {doc.get('workload')}, expected {workload_hash}")
            trace = ls.trace.deserialize_trace("\n".join(json.dumps(i) for i in doc["trace"]))
            lat = (Fraction(doc["latency_exact"]) if "latency_exact" in doc
                   else Fraction(doc["latency"]).limit_denominator(10 ** 12))
            out.append(ls.search.TuningRecord(trace, lat, np.array(doc["features"], dtype=np.float64),
                                              doc.get("hash", 0)))
    return out
