"""Scorer protocol and the batched GPU cost model (K7) + exact simulator (K8).

Reference functions replaced (all batched, one warp per program):
  * ``featurize(p, spec)``          `src/costmodel.py:21-79`   -> featurize_batch
  * ``CostModel.predict_features``  `src/costmodel.py:98-102`  -> score_batch
  * ``simulate_latency(p, spec)``   `src/machine.py:228-254`   -> sim_latency_batch
    (the parity-mode Runner: exact rationals, bit-identical to the reference)
"""

from __future__ import annotations

import ctypes
from fractions import Fraction
from typing import Protocol, Sequence

import numpy as np

from . import native
from .inputs import program_text


class Scorer(Protocol):
    def featurize_batch(self, programs, machine_spec=None) -> np.ndarray: ...

    def score_batch(self, features: np.ndarray, model) -> np.ndarray: ...


class AnalysisError(RuntimeError):
    pass


class GpuScorer:
    def __init__(self, device: int = 0):
        native.lib()
        self.device = device

    def analyze_arrays(self, texts: Sequence[str], machine_spec=None, model=None):
        """The batch in the reference Runner's own form, as arrays: exact
        latency numerators / denominators, features [n,9], predictions [n]
        (zeros without a model), per-program status -- the same outputs as the
        CPU reference arm's ``oracle.batch`` (one fused K7+K8 launch)."""
        n = len(texts)
        arr, lens, _keep = native.text_array(texts)
        spec = native.machine_spec_c(machine_spec)
        num = np.zeros(max(n, 1), np.int64)
        den = np.zeros(max(n, 1), np.int64)
        feats = np.zeros((max(n, 1), 9), np.float64)
        pred = np.zeros(max(n, 1), np.float64)
        status = np.zeros(max(n, 1), np.int32)
        mptr = ctypes.byref(native.linear_model_c(model)) if model is not None else None
        P = native.as_np_ptr
        native.check(native.lib().ls_analyze_batch(
            self.device, arr, lens, n, ctypes.byref(spec), mptr, P(num, ctypes.c_int64), P(den, ctypes.c_int64),
            P(feats, ctypes.c_double), P(pred, ctypes.c_double) if model is not None else None,
            P(status, ctypes.c_int32)), "ls_analyze_batch")
        return num[:n], den[:n], feats[:n], pred[:n], status[:n]

    def analyze(self, programs: Sequence, machine_spec=None, model=None,
                want_latency=True, want_features=True):
        """(latencies as Fractions or None, features [n,9] or None,
        predictions [n] or None) in one fused launch."""
        texts = [program_text(p) for p in programs]
        n = len(texts)
        arr, lens, _keep = native.text_array(texts)
        spec = native.machine_spec_c(machine_spec)
        num = np.zeros(max(n, 1), np.int64)
        den = np.zeros(max(n, 1), np.int64)
        feats = np.zeros((max(n, 1), 9), np.float64)
        pred = np.zeros(max(n, 1), np.float64)
        status = np.zeros(max(n, 1), np.int32)
        mptr = ctypes.byref(native.linear_model_c(model)) if model is not None else None
        P = native.as_np_ptr
        native.check(native.lib().ls_analyze_batch(
            self.device, arr, lens, n, ctypes.byref(spec), mptr,
            P(num, ctypes.c_int64) if want_latency else None,
            P(den, ctypes.c_int64) if want_latency else None,
            P(feats, ctypes.c_double) if (want_features or model is not None) else None,
            P(pred, ctypes.c_double) if model is not None else None,
            P(status, ctypes.c_int32)), "ls_analyze_batch")
        bad = np.nonzero(status[:n])[0]
        if len(bad):
            raise AnalysisError(f"{len(bad)} program(s) failed analysis "
                                f"(first index {bad[0]}, status {status[bad[0]]})")
        lats = [Fraction(int(a), int(b)) for a, b in zip(num[:n], den[:n])] if want_latency else None
        return lats, (feats[:n] if want_features else None), (pred[:n] if model is not None else None)

    def featurize_batch(self, programs, machine_spec=None) -> np.ndarray:
        return self.analyze(programs, machine_spec, want_latency=False)[1]

    def sim_latency_batch(self, programs, machine_spec=None) -> list:
        return self.analyze(programs, machine_spec, want_features=False)[0]

    def score_batch(self, features, model) -> np.ndarray:
        F = np.ascontiguousarray(np.asarray(features, dtype=np.float64).reshape(-1, 9))
        n = F.shape[0]
        out = np.zeros(max(n, 1), np.float64)
        native.check(native.lib().ls_score_batch(self.device, native.as_np_ptr(F, ctypes.c_double), n,
                                                 ctypes.byref(native.linear_model_c(model)),
                                                 native.as_np_ptr(out, ctypes.c_double)),
                     "ls_score_batch")
        return out[:n]


class DeviceBatch:
    """A population parsed, encoded and resident in HBM; `analyze()` runs the
    fused K7+K8 kernel only (the kernel-side timing path)."""

    def __init__(self, programs: Sequence, device: int = 0):
        texts = [program_text(p) for p in programs]
        self.n = len(texts)
        arr, lens, _keep = native.text_array(texts)
        h = ctypes.c_void_p()
        native.check(native.lib().ls_batch_create(device, arr, lens, self.n, ctypes.byref(h)),
                     "ls_batch_create")
        self._h = h

    def analyze(self, machine_spec=None, model=None, flags: int = 7) -> None:
        spec = native.machine_spec_c(machine_spec)
        mptr = ctypes.byref(native.linear_model_c(model)) if model is not None else None
        native.check(native.lib().ls_batch_analyze(self._h, ctypes.byref(spec), mptr, flags),
                     "ls_batch_analyze")

    def elapsed_ms(self) -> float:
        v = ctypes.c_float()
        native.check(native.lib().ls_batch_elapsed_ms(self._h, ctypes.byref(v)), "elapsed")
        return float(v.value)

    def results(self):
        n = max(self.n, 1)
        num, den = np.zeros(n, np.int64), np.zeros(n, np.int64)
        feats, pred = np.zeros((n, 9)), np.zeros(n)
        status = np.zeros(n, np.int32)
        P = native.as_np_ptr
        native.check(native.lib().ls_batch_results(self._h, P(num, ctypes.c_int64), P(den, ctypes.c_int64),
                                                   P(feats, ctypes.c_double), P(pred, ctypes.c_double),
                                                   P(status, ctypes.c_int32)), "ls_batch_results")
        return num[:self.n], den[:self.n], feats[:self.n], pred[:self.n], status[:self.n]

    def close(self):
        if getattr(self, "_h", None):
            native.lib().ls_batch_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
