"""Runner protocol and the B200 hardware runner.

The reference measures a candidate with ``simulate_latency`` inside
``_measure_batch(candidates, machine_spec, jobs)`` (`src/search.py:249-256`)
and prices the unscheduled program for the report's baseline
(`src/search.py:326`).  ``B200Runner`` keeps that exact call shape and return
type (a list of ``Fraction`` in candidate order) but instantiates every
candidate as an sm_100a kernel, runs it on the GPU, checks its output against
the reference output of the unscheduled program, and returns the measured
device time in nanoseconds as an exact ``Fraction`` (picosecond resolution),
so records, reports and ``load_records`` keep working unchanged.

Failures (illegal configuration, unsupported structure, launch failure,
parity failure, timeout) map to a finite sentinel latency --
``sentinel_factor`` x the baseline -- never ``inf``, because ``fit`` takes
``log(latency)`` (`src/costmodel.py:126`).
"""

from __future__ import annotations

import ctypes
from fractions import Fraction
from typing import Protocol, Sequence

import numpy as np

from . import native
from .inputs import program_text, random_inputs


class Runner(Protocol):
    def measure(self, candidates, machine_spec=None, jobs: int = 1) -> list: ...

    def baseline(self, e0, machine_spec=None) -> Fraction: ...


def ns_fraction(ns: float) -> Fraction:
    return Fraction(int(round(ns * 1000.0)), 1000)


class B200Runner:
    """Hardware runner on one GPU (one handle per device, not thread-safe)."""

    def __init__(self, device: int = 0, dtype: str = "bf16", min_repeats: int = 3,
                 max_repeats: int = 200, target_ms: float = 0.2, timeout_ms: float = 2.0,
                 rtol: float = 0.0, atol: float = 0.0, sentinel_factor: float = 1e4,
                 timeout_factor: float = 0.0, timeout_floor_ms: float = 0.05,
                 single_shot_factor: float = 0.0, carry_best: bool = False, flush_l2: bool = False,
                 baseline_timeout_factor: float = 0.0):
        L = native.lib()
        o = native.RunnerOptsC()
        o.dtype = 1 if dtype == "bf16" else 0
        o.min_repeats, o.max_repeats = min_repeats, max_repeats
        o.target_ms, o.timeout_ms = target_ms, timeout_ms
        o.rtol, o.atol = rtol, atol
        o.timeout_factor, o.timeout_floor_ms = timeout_factor, timeout_floor_ms
        o.single_shot_factor = single_shot_factor
        o.carry_best = 1 if carry_best else 0
        o.flush_l2 = 1 if flush_l2 else 0  # cold-L2 timing of every repeat
        h = ctypes.c_void_p()
        native.check(L.ls_runner_create(device, ctypes.byref(o), ctypes.byref(h)),
                     "ls_runner_create")
        self._h = h
        self.device = device
        self.dtype = dtype
        self.sentinel_factor = sentinel_factor
        # > 0: once the e0 baseline is measured, the deadline cap becomes
        # max(timeout_floor_ms, factor x baseline) (the bench's own policy:
        # a candidate slower than 2x the unscheduled program is aborted)
        self.baseline_timeout_factor = baseline_timeout_factor
        self.timeout_floor_ms = timeout_floor_ms
        self.timeout_ms = timeout_ms
        self.e0_json = None
        self._baseline = None
        self.last_results: list = []

    def close(self):
        if getattr(self, "_h", None):
            native.lib().ls_runner_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- workload -------------------------------------------------------------
    def set_workload(self, e0, inputs: dict | None = None, seed: int = 0) -> None:
        """Upload the workload inputs once (the reference's random_inputs by
        default).  ``inputs`` maps input-buffer names to arrays."""
        e0_json = program_text(e0)
        import json
        names = [b["name"] for b in json.loads(e0_json)["buffers"] if b["role"] == "input"]
        if inputs is None:
            inputs = random_inputs(e0_json, seed)
        arrs = [np.ascontiguousarray(np.asarray(inputs[n], dtype=np.float32)) for n in names]
        ptrs = (native.c_f32p * len(arrs))(*[native.as_np_ptr(a, ctypes.c_float) for a in arrs])
        b = e0_json.encode()
        native.check(native.lib().ls_runner_set_workload(self._h, b, len(b), ptrs, len(arrs)),
                     "ls_runner_set_workload")
        self.e0_json = e0_json
        self._baseline = None
        if self.baseline_timeout_factor > 0:  # back to the configured cap until e0 is re-measured
            native.check(native.lib().ls_runner_set_timeout(self._h, self.timeout_ms), "ls_runner_set_timeout")

    # -- measurement ----------------------------------------------------------
    def measure_programs(self, programs: Sequence) -> list:
        """Raw per-candidate results (status, family, config, ns, parity)."""
        texts = [program_text(p) for p in programs]
        arr, lens, _keep = native.text_array(texts)
        n = len(texts)
        res = (native.ResultC * max(n, 1))()
        native.check(native.lib().ls_runner_measure(self._h, arr, lens, n, res),
                     "ls_runner_measure")
        self.last_results = native.results_to_dicts(res, n)
        return self.last_results

    def plan_programs(self, programs: Sequence) -> list:
        texts = [program_text(p) for p in programs]
        arr, lens, _keep = native.text_array(texts)
        n = len(texts)
        res = (native.ResultC * max(n, 1))()
        native.check(native.lib().ls_runner_plan(self._h, arr, lens, n, res), "ls_runner_plan")
        return native.results_to_dicts(res, n)

    def baseline_result(self) -> dict:
        res = (native.ResultC * 1)()
        native.check(native.lib().ls_runner_baseline(self._h, res), "ls_runner_baseline")
        return native.results_to_dicts(res, 1)[0]

    def baseline(self, e0=None, machine_spec=None) -> Fraction:
        """Measured latency of the unscheduled program (`src/search.py:326`)."""
        if e0 is not None and program_text(e0) != self.e0_json:
            self.set_workload(e0)
        if self._baseline is None:
            r = self.baseline_result()
            if r["status"] != "OK":
                raise native.NativeError(f"baseline e0 failed to run: {r['status']}")
            self._baseline = ns_fraction(r["latency_ns"])
            if self.baseline_timeout_factor > 0:
                cap = max(self.timeout_floor_ms, self.baseline_timeout_factor * r["latency_ns"] / 1e6)
                native.check(native.lib().ls_runner_set_timeout(self._h, cap), "ls_runner_set_timeout")
        return self._baseline

    def sentinel(self) -> Fraction:
        return self.baseline() * Fraction(self.sentinel_factor)

    def latencies(self, results) -> list:
        """OK -> measured ns; TIMEOUT -> the abort time (a lower bound, still
        ordered below every failure); anything else -> the finite sentinel."""
        out = []
        for r in results:
            if r["status"] == "OK":
                out.append(ns_fraction(r["latency_ns"]))
            elif r["status"] == "TIMEOUT" and r["latency_ns"] > 0:
                out.append(min(ns_fraction(r["latency_ns"]), self.sentinel()))
            else:
                out.append(self.sentinel())
        return out

    def measure(self, candidates, machine_spec=None, jobs: int = 1) -> list:
        """`_measure_batch` signature: latencies in candidate order."""
        return self.latencies(self.measure_programs(candidates))

    def elapsed_ms(self) -> float:
        v = ctypes.c_float()
        native.check(native.lib().ls_runner_elapsed_ms(self._h, ctypes.byref(v)), "elapsed")
        return float(v.value)

    def launch_count(self) -> int:
        v = ctypes.c_int64()
        native.check(native.lib().ls_runner_launch_count(self._h, ctypes.byref(v)), "launches")
        return int(v.value)

    def trace_tc(self, program, launches: int = 1, max_ctas: int = 1 << 15) -> np.ndarray:
        """Per-CTA ``%globaltimer`` stamps of a tcgen05 GEMM / conv candidate
        (``ls_runner_trace_tc``): [launches * n_ctas, 8] int64 ns -- start,
        setup done, first stage landed, accumulator done, partial staged,
        zeroing flag acquired, stored, smid."""
        b = program_text(program).encode()
        buf = (ctypes.c_uint64 * (8 * max_ctas))()
        n = ctypes.c_int()
        native.check(native.lib().ls_runner_trace_tc(self._h, b, len(b), launches, buf, max_ctas,
                                                     ctypes.byref(n)), "ls_runner_trace_tc")
        return np.frombuffer(buf, dtype=np.uint64).reshape(-1, 8)[: n.value * launches].astype(np.int64)

    def kernel_span_us(self, program, samples: int = 5) -> float:
        """Device-side duration of ONE isolated launch of a tcgen05 candidate:
        first CTA start to last CTA end (globaltimer), median of ``samples``
        single-launch traces -- the kernel without the host/driver launch
        latency that CUDA events around a lone launch also include."""
        spans = []
        for _ in range(samples):
            a = self.trace_tc(program, 1)
            spans.append((a[:, 6].max() - a[:, 0].min()) / 1e3)
        return float(np.median(spans))

    def debug_stats(self, launch_host_us: float = 0.0) -> dict:
        a = np.zeros(8, np.float64)
        a[7] = launch_host_us
        native.check(native.lib().ls_runner_debug_stats(self._h, native.as_np_ptr(a, ctypes.c_double), 8),
                     "debug_stats")
        return {"phase_a_host_ms": a[0], "phase_b_host_ms": a[1], "spin_us": a[2], "empty_candidate_us": a[4],
                "device_best_us": a[5], "phase_a_enqueue_ms": a[6], "plan_ms": a[3]}

    def last_output(self) -> np.ndarray:
        import json
        doc = json.loads(self.e0_json)
        out = [b for b in doc["buffers"] if b["role"] == "output"][0]
        n = int(np.prod(out["shape"]))
        a = np.empty(n, dtype=np.float32)
        native.check(native.lib().ls_runner_last_output(self._h, native.as_np_ptr(a, ctypes.c_float), n),
                     "last_output")
        return a.reshape(out["shape"])

    def reference_output(self) -> np.ndarray:
        import json
        doc = json.loads(self.e0_json)
        out = [b for b in doc["buffers"] if b["role"] == "output"][0]
        n = int(np.prod(out["shape"]))
        a = np.empty(n, dtype=np.float64)
        native.check(native.lib().ls_runner_reference_output(self._h, native.as_np_ptr(a, ctypes.c_double), n),
                     "reference_output")
        return a.reshape(out["shape"])
