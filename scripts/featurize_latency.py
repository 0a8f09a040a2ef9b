"""Latency of one-program featurize calls (the reference search's access
pattern: one K7 call per new program) vs the batched call, on the B200."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from conftest import load_population  # noqa: E402
from paper_2205_13603_b200.scorer import DeviceBatch, GpuScorer  # noqa: E402

hdr, pop = load_population("gmm512")
texts = [p["program"] for p in pop[:512]]
s = GpuScorer(0)
s.featurize_batch(texts[:4])
for name, fn in (("featurize_batch([1])", lambda t: s.featurize_batch([t])),
                 ("analyze_arrays([1]) features+latency", lambda t: s.analyze_arrays([t]))):
    t0 = time.perf_counter()
    for t in texts[:200]:
        fn(t)
    print(f"{name}: {(time.perf_counter() - t0) / 200 * 1e6:.1f} us per call")
t0 = time.perf_counter()
s.featurize_batch(texts)
print(f"featurize_batch(512): {(time.perf_counter() - t0) * 1e6 / 512:.2f} us per program")
b = DeviceBatch(texts[:1])
for flags, what in ((2, "features"), (1, "latency"), (7, "all")):
    b.analyze(flags=flags)
    ms = []
    for _ in range(50):
        b.analyze(flags=flags)
        ms.append(b.elapsed_ms())
    ms.sort()
    print(f"device time, 1 program, {what}: {ms[len(ms) // 2] * 1e3:.1f} us")
