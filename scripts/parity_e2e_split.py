"""Where the parity-mode end-to-end call (ls_analyze_batch from host program
texts, the like-for-like counterpart of the reference arm) spends its time
for a 1024-program BERT-FFN slice: Python marshalling, the native call
(host parse + encode on the host pool, one H2D, K7+K8, one D2H), and the
kernel alone."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from conftest import load_model, load_population  # noqa: E402
from paper_2205_13603_b200 import native  # noqa: E402
from paper_2205_13603_b200.scorer import DeviceBatch, GpuScorer  # noqa: E402

hdr, pop = load_population(sys.argv[1] if len(sys.argv) > 1 else "bert_ffn")
texts = [p["program"] for p in pop[:1024]]
model = load_model()
s = GpuScorer(0)
s.analyze_arrays(texts, model=model)
N = 20
t0 = time.perf_counter()
for _ in range(N):
    s.analyze_arrays(texts, model=model)
full = (time.perf_counter() - t0) / N
t0 = time.perf_counter()
for _ in range(N):
    native.text_array(texts)
marsh = (time.perf_counter() - t0) / N
b = DeviceBatch(texts)
b.analyze(model=model)
ks = []
for _ in range(N):
    b.analyze(model=model)
    ks.append(b.elapsed_ms())
print(f"analyze_arrays(1024): {full * 1e3:.2f} ms = {1024 / full / 1e3:.0f} k programs/s; "
      f"text marshalling {marsh * 1e3:.2f} ms; K7+K8 device {min(ks):.3f} ms; host threads {os.cpu_count()}")
