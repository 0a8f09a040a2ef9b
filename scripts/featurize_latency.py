"""Latency of one-program featurize calls (the reference search's access pattern)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
from conftest import load_population
from paper_2205_13603_b200.scorer import GpuScorer
hdr, pop = load_population("bert_ffn")
texts = [p["program"] for p in pop[:400]]
s = GpuScorer(0)
s.featurize_batch(texts[:8])
t0 = time.perf_counter()
for t in texts[:300]:
    s.featurize_batch([t])
dt = (time.perf_counter() - t0) / 300
t0 = time.perf_counter()
s.featurize_batch(texts)
db = time.perf_counter() - t0
print(f"one-program featurize: {dt*1e6:.1f} us/call; batch of {len(texts)}: {db*1e3:.2f} ms")
