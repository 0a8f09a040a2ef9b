"""Run the fused K7+K8 kernel on a device-resident population (for ncu)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from conftest import load_model, load_population  # noqa: E402
from paper_2205_13603_b200.scorer import DeviceBatch  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "bert_ffn"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
hdr, pop = load_population(name)
model = load_model()
b = DeviceBatch([p["program"] for p in pop[:n]])
ms = []
for _ in range(reps):
    b.analyze(model=model)
    ms.append(b.elapsed_ms())
blob_words = None
print(json.dumps({"programs": n, "ms": ms, "programs_per_s": n / (min(ms) / 1e3)}))
