"""Population measurement sharded across the GPUs of one box.

One worker process per GPU (``CUDA_VISIBLE_DEVICES`` pinned, spawn start
method), each holding its own ``B200Runner`` with the workload uploaded once.
``ShardedRunner.measure`` deals the ordered batch round-robin by index, every
worker measures its slice on its own stream, and the host reassembles results
in candidate order.  There is no collective: candidates are
independent, so the only exchange is the host-side gather.
"""

from __future__ import annotations

import multiprocessing as mp
import os
from fractions import Fraction

from .inputs import program_text


def deal(n: int, workers: int):
    """Round-robin index slices: worker w gets [w, w+W, w+2W, ...]."""
    return [list(range(w, n, workers)) for w in range(workers)]


def _fake_result(text: str) -> dict:
    # deterministic stand-in used by the CPU tests of the sharding logic
    import zlib
    return {"status": "OK", "family": "fake", "repeats": 1, "cfg": [0] * 13,
            "latency_ns": 1000.0 + zlib.crc32(text.encode()) % 9000, "max_abs_err": 0.0, "mismatches": 0}


def _worker(conn, device: int, backend: str, opts: dict):
    if backend == "b200":
        os.environ["CUDA_VISIBLE_DEVICES"] = str(device)
        from .runner import B200Runner
        runner = B200Runner(device=0, **opts)
    else:
        runner = None
    try:
        while True:
            cmd, payload = conn.recv()
            if cmd == "close":
                break
            try:
                if cmd == "workload":
                    if runner is not None:
                        e0, inputs = payload
                        runner.set_workload(e0, inputs)
                    conn.send(("ok", None))
                elif cmd == "measure":
                    if runner is None:
                        conn.send(("ok", [_fake_result(t) for t in payload]))
                    else:
                        res = runner.measure_programs(payload)
                        conn.send(("ok", (res, runner.elapsed_ms(), runner.launch_count())))
                elif cmd == "baseline":
                    conn.send(("ok", _fake_result("e0") if runner is None else runner.baseline_result()))
                else:
                    conn.send(("err", f"unknown command {cmd}"))
            except Exception as exc:  # report, keep serving
                conn.send(("err", repr(exc)))
    finally:
        if runner is not None:
            runner.close()
        conn.close()


class ShardedRunner:
    """Runner protocol over N GPUs (one process each)."""

    def __init__(self, devices, backend: str = "b200", sentinel_factor: float = 1e4, **opts):
        self.devices = list(devices)
        self.backend = backend
        self.sentinel_factor = sentinel_factor
        ctx = mp.get_context("spawn")
        self._conns, self._procs = [], []
        for d in self.devices:
            a, b = ctx.Pipe()
            p = ctx.Process(target=_worker, args=(b, d, backend, opts), daemon=True)
            p.start()
            self._conns.append(a)
            self._procs.append(p)
        self._baseline = None
        self.last_device_ms = []
        self.last_results = []

    def _call_all(self, cmd, payloads):
        for c, pl in zip(self._conns, payloads):
            c.send((cmd, pl))
        out = []
        for c in self._conns:
            st, val = c.recv()
            if st != "ok":
                raise RuntimeError(f"worker failed: {val}")
            out.append(val)
        return out

    def set_workload(self, e0, inputs=None) -> None:
        self._call_all("workload", [(program_text(e0), inputs)] * len(self._conns))
        self._baseline = None

    def measure_programs(self, programs) -> list:
        texts = [program_text(p) for p in programs]
        slices = deal(len(texts), len(self._conns))
        vals = self._call_all("measure", [[texts[i] for i in sl] for sl in slices])
        out = [None] * len(texts)
        self.last_device_ms = []
        for sl, v in zip(slices, vals):
            res = v if self.backend != "b200" else v[0]
            if self.backend == "b200":
                self.last_device_ms.append(v[1])
            for i, r in zip(sl, res):
                out[i] = r
        self.last_results = out
        return out

    def baseline(self, e0=None, machine_spec=None) -> Fraction:
        if e0 is not None:
            self.set_workload(e0)
        if self._baseline is None:
            st, r = None, None
            self._conns[0].send(("baseline", None))
            st, r = self._conns[0].recv()
            if st != "ok" or r["status"] != "OK":
                raise RuntimeError(f"baseline failed: {r}")
            self._baseline = Fraction(int(round(r["latency_ns"] * 1000)), 1000)
        return self._baseline

    def measure(self, candidates, machine_spec=None, jobs: int = 1) -> list:
        res = self.measure_programs(candidates)
        sentinel = self.baseline() * Fraction(self.sentinel_factor)
        out = []
        for r in res:
            if r["status"] == "OK":
                out.append(Fraction(int(round(r["latency_ns"] * 1000)), 1000))
            elif r["status"] == "TIMEOUT" and r["latency_ns"] > 0:
                out.append(min(Fraction(int(round(r["latency_ns"] * 1000)), 1000), sentinel))
            else:
                out.append(sentinel)
        return out

    def close(self):
        for c in self._conns:
            try:
                c.send(("close", None))
            except Exception:
                pass
        for p in self._procs:
            p.join(timeout=10)
        self._conns, self._procs = [], []

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
