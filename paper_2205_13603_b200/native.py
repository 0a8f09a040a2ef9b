"""ctypes binding of the C ABI in ``include/loopsched_b200.h``.

The shared library ``_lib/libls_b200.so`` is built in-tree by
``__graft_entry__.build()`` (``make -C paper_2205_13603_b200/csrc``).  Loading
fails loudly when it is missing -- there is no CPU fallback for any compute
entry point.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from fractions import Fraction

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# LSB_LIB_PATH: an alternative build of the same library (A/B experiments)
LIB_PATH = os.environ.get("LSB_LIB_PATH") or os.path.join(HERE, "_lib", "libls_b200.so")
CSRC = os.path.join(HERE, "csrc")

c_i64p = ctypes.POINTER(ctypes.c_int64)
c_i32p = ctypes.POINTER(ctypes.c_int32)
c_f64p = ctypes.POINTER(ctypes.c_double)
c_f32p = ctypes.POINTER(ctypes.c_float)


class MachineSpecC(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int64) for n in
                ("cores", "vector_lanes", "cache_capacity", "hit_cost", "miss_cost",
                 "flop_cost", "tensor_unit_cost", "unroll_num", "unroll_den")]


class LinearModelC(ctypes.Structure):
    _fields_ = [("w", ctypes.c_double * 9), ("mean", ctypes.c_double * 9),
                ("scale", ctypes.c_double * 9), ("intercept", ctypes.c_double),
                ("n_records", ctypes.c_int64), ("is_fit", ctypes.c_int32)]


class RunnerOptsC(ctypes.Structure):
    _fields_ = [("dtype", ctypes.c_int32), ("min_repeats", ctypes.c_int32),
                ("max_repeats", ctypes.c_int32), ("target_ms", ctypes.c_double),
                ("timeout_ms", ctypes.c_double), ("rtol", ctypes.c_double),
                ("atol", ctypes.c_double), ("flush_l2", ctypes.c_int32),
                ("carry_best", ctypes.c_int32), ("timeout_factor", ctypes.c_double),
                ("timeout_floor_ms", ctypes.c_double), ("single_shot_factor", ctypes.c_double)]


class ResultC(ctypes.Structure):
    _fields_ = [("status", ctypes.c_int32), ("family", ctypes.c_int32),
                ("repeats", ctypes.c_int32), ("cfg", ctypes.c_int32 * 13),
                ("latency_ns", ctypes.c_double), ("max_abs_err", ctypes.c_double),
                ("mismatches", ctypes.c_int64), ("checked_ns", ctypes.c_double)]


class ReplayResultC(ctypes.Structure):
    _fields_ = [("status", ctypes.c_int32), ("index", ctypes.c_int32), ("hash", ctypes.c_uint64),
                ("program", ctypes.c_void_p), ("trace", ctypes.c_void_p), ("reason", ctypes.c_void_p)]


EXPORTS = {
    # name: (restype, argtypes)
    "ls_sim_latency_batch": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(ctypes.c_char_p),
                                            ctypes.POINTER(ctypes.c_size_t), ctypes.c_int,
                                            ctypes.POINTER(MachineSpecC), c_i64p, c_i64p, c_i32p]),
    "ls_featurize_batch": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(ctypes.c_char_p),
                                          ctypes.POINTER(ctypes.c_size_t), ctypes.c_int,
                                          ctypes.POINTER(MachineSpecC), c_f64p, c_i32p]),
    "ls_score_batch": (ctypes.c_int, [ctypes.c_int, c_f64p, ctypes.c_int,
                                      ctypes.POINTER(LinearModelC), c_f64p]),
    "ls_analyze_batch": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(ctypes.c_char_p),
                                        ctypes.POINTER(ctypes.c_size_t), ctypes.c_int,
                                        ctypes.POINTER(MachineSpecC), ctypes.POINTER(LinearModelC),
                                        c_i64p, c_i64p, c_f64p, c_f64p, c_i32p]),
    "ls_batch_create": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(ctypes.c_char_p),
                                       ctypes.POINTER(ctypes.c_size_t), ctypes.c_int,
                                       ctypes.POINTER(ctypes.c_void_p)]),
    "ls_batch_analyze": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(MachineSpecC),
                                        ctypes.POINTER(LinearModelC), ctypes.c_int]),
    "ls_batch_results": (ctypes.c_int, [ctypes.c_void_p, c_i64p, c_i64p, c_f64p, c_f64p, c_i32p]),
    "ls_batch_elapsed_ms": (ctypes.c_int, [ctypes.c_void_p, c_f32p]),
    "ls_batch_destroy": (None, [ctypes.c_void_p]),
    "ls_runner_create": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(RunnerOptsC),
                                        ctypes.POINTER(ctypes.c_void_p)]),
    "ls_runner_set_workload": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_char_p, ctypes.c_size_t,
                                              ctypes.POINTER(c_f32p), ctypes.c_int]),
    "ls_runner_measure": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_char_p),
                                         ctypes.POINTER(ctypes.c_size_t), ctypes.c_int,
                                         ctypes.POINTER(ResultC)]),
    "ls_runner_baseline": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ResultC)]),
    "ls_runner_plan": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_char_p),
                                      ctypes.POINTER(ctypes.c_size_t), ctypes.c_int,
                                      ctypes.POINTER(ResultC)]),
    "ls_plan_programs": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_size_t,
                                        ctypes.POINTER(ctypes.c_char_p),
                                        ctypes.POINTER(ctypes.c_size_t), ctypes.c_int,
                                        ctypes.c_int32, ctypes.POINTER(ResultC)]),
    "ls_runner_last_output": (ctypes.c_int, [ctypes.c_void_p, c_f32p, ctypes.c_size_t]),
    "ls_runner_reference_output": (ctypes.c_int, [ctypes.c_void_p, c_f64p, ctypes.c_size_t]),
    "ls_runner_elapsed_ms": (ctypes.c_int, [ctypes.c_void_p, c_f32p]),
    "ls_runner_launch_count": (ctypes.c_int, [ctypes.c_void_p, c_i64p]),
    "ls_runner_debug_stats": (ctypes.c_int, [ctypes.c_void_p, c_f64p, ctypes.c_int]),
    "ls_runner_set_timeout": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_double]),
    "ls_runner_trace_tc": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_char_p, ctypes.c_size_t, ctypes.c_int,
                                          ctypes.POINTER(ctypes.c_uint64), ctypes.c_int, c_i32p]),
    "ls_runner_destroy": (None, [ctypes.c_void_p]),
    "ls_replayer_create": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_size_t, ctypes.POINTER(ctypes.c_void_p)]),
    "ls_replayer_hash": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_uint64)]),
    "ls_replay_batch": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_char_p),
                                       ctypes.POINTER(ctypes.c_size_t), ctypes.c_int,
                                       ctypes.POINTER(ReplayResultC)]),
    "ls_replay_resample": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_char_p, ctypes.c_size_t, ctypes.c_uint64,
                                          ctypes.POINTER(ReplayResultC)]),
    "ls_replay_free": (None, [ctypes.POINTER(ReplayResultC), ctypes.c_int]),
    "ls_replayer_destroy": (None, [ctypes.c_void_p]),
    "ls_replay_neighbours": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_char_p),
                                            ctypes.POINTER(ctypes.c_size_t), ctypes.c_int,
                                            ctypes.POINTER(ctypes.c_void_p)]),
    "ls_neighbours_count": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_int)]),
    "ls_neighbours_get": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.POINTER(ctypes.c_uint64),
                                         ctypes.POINTER(ctypes.c_char_p)]),
    "ls_neighbours_stats": (ctypes.c_int, [ctypes.c_void_p, c_i64p]),
    "ls_neighbours_destroy": (None, [ctypes.c_void_p]),
    "ls_program_hash": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_size_t, ctypes.POINTER(ctypes.c_uint64)]),
    "ls_last_error": (ctypes.c_char_p, []),
    "ls_version": (ctypes.c_char_p, []),
}

STATUS = {0: "OK", 1: "ILLEGAL", 2: "UNSUPPORTED", 3: "PARSE", 4: "LAUNCH", 5: "PARITY",
          6: "TIMEOUT"}
FAMILY = {0: "none", 1: "naive", 2: "simt", 3: "tcgen05", 4: "loopnest", 5: "generic", 6: "nestgen",
          7: "simt_affine", 8: "tcgen05_conv", 9: "affcopy"}


class NativeError(RuntimeError):
    pass


def build(verbose: bool = False) -> str:
    jobs = str(max(1, min(8, os.cpu_count() or 1)))
    subprocess.run(["make", "-s", "-j", jobs, "-C", CSRC], check=True,
                   stdout=None if verbose else subprocess.DEVNULL)
    return LIB_PATH


_lib = None


def lib():
    """The loaded library; raises when it was never built (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise NativeError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                              "(the B200 path has no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in EXPORTS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(status: int, what: str) -> None:
    if status != 0:
        msg = lib().ls_last_error().decode(errors="replace")
        raise NativeError(f"{what} failed (status {status}): {msg}")


def text_array(programs):
    """(const char* const*, const size_t*, keep-alive) for a list of program /
    trace texts.  Large batches are joined into one buffer and the pointer
    array is built with numpy (creating one ``c_char_p`` per text costs more
    than the native call's parsing for 1k programs); texts must then be ASCII
    (the reference writes JSON with ``ensure_ascii``), else per-text encoding."""
    n = len(programs)
    if n >= 64 and all(isinstance(p, str) for p in programs):
        lens = np.fromiter(map(len, programs), dtype=np.uint64, count=n)
        try:
            b = "".join(programs).encode("ascii")
        except UnicodeEncodeError:
            b = None
        if b is not None:
            buf = np.frombuffer(b, dtype=np.uint8)
            off = np.zeros(n, dtype=np.uint64)
            np.cumsum(lens[:-1], out=off[1:])
            ptrs = off + np.uint64(buf.ctypes.data)
            return (ptrs.ctypes.data_as(ctypes.POINTER(ctypes.c_char_p)),
                    lens.ctypes.data_as(ctypes.POINTER(ctypes.c_size_t)), (b, buf, ptrs, lens))
    enc = [p.encode() if isinstance(p, str) else bytes(p) for p in programs]
    arr = (ctypes.c_char_p * max(n, 1))(*enc)
    lens = (ctypes.c_size_t * max(n, 1))(*[len(b) for b in enc])
    return arr, lens, enc


_SPEC_CACHE: dict = {}


def machine_spec_c(spec=None) -> MachineSpecC:
    """From a reference MachineSpec, a dict, or None (defaults of
    `src/machine.py:22-31`); memoized for hashable specs (the search passes
    the same frozen MachineSpec on every call)."""
    try:
        hit = _SPEC_CACHE.get(spec)
    except TypeError:
        return _machine_spec_c(spec)
    if hit is None:
        hit = _SPEC_CACHE[spec] = _machine_spec_c(spec)
    return hit


def _machine_spec_c(spec=None) -> MachineSpecC:
    d = {"cores": 4, "vector_lanes": 8, "cache_capacity": 4096, "hit_cost": 1,
         "miss_cost": 8, "flop_cost": 1, "unroll_discount": 0.9, "tensor_unit_cost": 8}
    if spec is not None:
        src = spec if isinstance(spec, dict) else spec.to_json()
        d.update(src)
    disc = Fraction(str(d["unroll_discount"]))
    return MachineSpecC(d["cores"], d["vector_lanes"], d["cache_capacity"], d["hit_cost"],
                        d["miss_cost"], d["flop_cost"], d["tensor_unit_cost"],
                        disc.numerator, disc.denominator)


def linear_model_c(model) -> LinearModelC:
    """From a reference CostModel or a dict with the same field names."""
    get = (lambda k, dflt=None: model.get(k, dflt)) if isinstance(model, dict) \
        else (lambda k, dflt=None: getattr(model, k, dflt))
    m = LinearModelC()
    w = get("weights")
    m.is_fit = 1 if w is not None else 0
    if w is not None:
        mean, scale = get("feature_mean"), get("feature_scale")
        for i in range(9):
            m.w[i] = float(w[i])
            m.mean[i] = float(mean[i])
            m.scale[i] = float(scale[i])
    m.intercept = float(get("intercept", 0.0) or 0.0)
    m.n_records = int(get("n_records", 0) or 0)
    return m


_RESULT_DTYPE = np.dtype([("status", np.int32), ("family", np.int32), ("repeats", np.int32),
                          ("cfg", np.int32, (13,)), ("latency_ns", np.float64), ("max_abs_err", np.float64),
                          ("mismatches", np.int64), ("checked_ns", np.float64)], align=True)


def results_to_dicts(res, n):
    """ls_result[n] -> dicts, column-wise through numpy (per-field ctypes
    access cost ~3 us per candidate)."""
    if n <= 0:
        return []
    if _RESULT_DTYPE.itemsize != ctypes.sizeof(ResultC):
        raise RuntimeError("ls_result layout mismatch")
    a = np.frombuffer(res, dtype=_RESULT_DTYPE, count=n)
    st, fam, rep = a["status"].tolist(), a["family"].tolist(), a["repeats"].tolist()
    cfg, lat = a["cfg"].tolist(), a["latency_ns"].tolist()
    err, mis = a["max_abs_err"].tolist(), a["mismatches"].tolist()
    chk = a["checked_ns"].tolist()
    return [{"status": STATUS.get(st[i], str(st[i])), "family": FAMILY.get(fam[i], "?"), "repeats": rep[i],
             "cfg": cfg[i], "latency_ns": lat[i], "max_abs_err": err[i], "mismatches": mis[i],
             "checked_ns": chk[i]}
            for i in range(n)]


def plan_programs(e0: str, programs, dtype: str = "bf16"):
    """Host-only instantiation of each program (no GPU needed)."""
    arr, lens, _keep = text_array(programs)
    n = len(programs)
    res = (ResultC * max(n, 1))()
    e = e0.encode()
    check(lib().ls_plan_programs(e, len(e), arr, lens, n, 1 if dtype == "bf16" else 0, res),
          "ls_plan_programs")
    return results_to_dicts(res, n)


def as_np_ptr(a: np.ndarray, ctype):
    return a.ctypes.data_as(ctypes.POINTER(ctype))
