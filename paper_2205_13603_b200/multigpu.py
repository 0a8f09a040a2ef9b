"""Population measurement sharded across the GPUs of one box.

One worker process per GPU (``CUDA_VISIBLE_DEVICES`` pinned, spawn start
method), each holding its own ``B200Runner`` with the workload uploaded once.
``ShardedRunner.measure`` deals the ordered batch round-robin by index, every
worker measures its slice on its own stream, and the host reassembles results
in candidate order.  There is no collective: candidates are
independent, so the only exchange is the host-side gather.  This replaces the
reference's thread pool over one batch (`src/search.py:249-256`).

Each request carries a sequence number and every worker's reply is read
before any error is raised, so a failed call never leaves a stale reply in a
pipe for the next call to pick up.
"""

from __future__ import annotations

import multiprocessing as mp
import os
from fractions import Fraction

from .inputs import program_text


def deal(n: int, workers: int):
    """Round-robin index slices: worker w gets [w, w+W, w+2W, ...]."""
    return [list(range(w, n, workers)) for w in range(workers)]


def b200_factory(device: int, **opts):
    """The production worker runner: a ``B200Runner`` on the pinned device."""
    os.environ["CUDA_VISIBLE_DEVICES"] = str(device)
    from .runner import B200Runner
    return B200Runner(device=0, **opts)


def _worker(conn, device: int, factory, opts: dict):
    runner = factory(device, **opts)
    try:
        while True:
            seq, cmd, payload = conn.recv()
            if cmd == "close":
                break
            try:
                if cmd == "workload":
                    e0, inputs = payload
                    runner.set_workload(e0, inputs)
                    conn.send((seq, "ok", None))
                elif cmd == "measure":
                    res = runner.measure_programs(payload)
                    conn.send((seq, "ok", (res, runner.elapsed_ms(), runner.launch_count())))
                elif cmd == "baseline":
                    conn.send((seq, "ok", runner.baseline_result()))
                else:
                    conn.send((seq, "err", f"unknown command {cmd}"))
            except Exception as exc:  # report, keep serving
                conn.send((seq, "err", repr(exc)))
    finally:
        close = getattr(runner, "close", None)
        if close is not None:
            close()
        conn.close()


def ns_fraction(ns: float) -> Fraction:
    return Fraction(int(round(ns * 1000.0)), 1000)


class ShardedRunner:
    """Runner protocol over N GPUs (one process each).  ``factory(device,
    **opts)`` builds each worker's runner inside the worker process (default:
    a ``B200Runner`` pinned to that GPU)."""

    def __init__(self, devices, factory=b200_factory, sentinel_factor: float = 1e4, **opts):
        self.devices = list(devices)
        self.sentinel_factor = sentinel_factor
        ctx = mp.get_context("spawn")
        self._conns, self._procs = [], []
        for d in self.devices:
            a, b = ctx.Pipe()
            p = ctx.Process(target=_worker, args=(b, d, factory, opts), daemon=True)
            p.start()
            self._conns.append(a)
            self._procs.append(p)
        self._seq = 0
        self._e0_text = None
        self._baseline = None
        self.last_device_ms = []
        self.last_results = []

    def _call(self, conns, cmd, payloads):
        """Send one request per connection, then read EVERY reply (matched by
        sequence number) before raising on any worker error."""
        self._seq += 1
        seq = self._seq
        for c, pl in zip(conns, payloads):
            c.send((seq, cmd, pl))
        out, errs = [], []
        for w, c in enumerate(conns):
            while True:
                rseq, st, val = c.recv()
                if rseq == seq:
                    break  # an older reply can only be left by an interrupted call: drop it
            if st != "ok":
                errs.append(f"worker {w} (device {self.devices[w]}): {val}")
            out.append(val)
        if errs:
            raise RuntimeError("worker failed: " + "; ".join(errs))
        return out

    def set_workload(self, e0, inputs=None) -> None:
        text = program_text(e0)
        self._call(self._conns, "workload", [(text, inputs)] * len(self._conns))
        self._e0_text = text
        self._baseline = None

    def measure_programs(self, programs) -> list:
        texts = [program_text(p) for p in programs]
        slices = deal(len(texts), len(self._conns))
        vals = self._call(self._conns, "measure", [[texts[i] for i in sl] for sl in slices])
        out = [None] * len(texts)
        self.last_device_ms = []
        for sl, (res, dev_ms, _launches) in zip(slices, vals):
            self.last_device_ms.append(dev_ms)
            for i, r in zip(sl, res):
                out[i] = r
        self.last_results = out
        return out

    def baseline(self, e0=None, machine_spec=None) -> Fraction:
        """Measured e0 latency on worker 0; the workload (and any custom
        inputs) is re-uploaded only when ``e0`` differs from the loaded one."""
        if e0 is not None and program_text(e0) != self._e0_text:
            self.set_workload(e0)
        if self._baseline is None:
            r, = self._call(self._conns[:1], "baseline", [None])
            if r["status"] != "OK":
                raise RuntimeError(f"baseline failed: {r}")
            self._baseline = ns_fraction(r["latency_ns"])
        return self._baseline

    def measure(self, candidates, machine_spec=None, jobs: int = 1) -> list:
        res = self.measure_programs(candidates)
        sentinel = self.baseline() * Fraction(self.sentinel_factor)
        out = []
        for r in res:
            if r["status"] == "OK":
                out.append(ns_fraction(r["latency_ns"]))
            elif r["status"] == "TIMEOUT" and r["latency_ns"] > 0:
                out.append(min(ns_fraction(r["latency_ns"]), sentinel))
            else:
                out.append(sentinel)
        return out

    def close(self):
        for c in self._conns:
            try:
                c.send((0, "close", None))
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
