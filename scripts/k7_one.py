"""One-program K7 launches (features only, the search's access pattern) on a
device-resident program, for ncu source-level captures:
  ncu --set full --import-source on -k regex:analyze -c 1 python scripts/k7_one.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from conftest import load_population  # noqa: E402
from paper_2205_13603_b200.scorer import DeviceBatch  # noqa: E402

hdr, pop = load_population(sys.argv[1] if len(sys.argv) > 1 else "gmm512")
b = DeviceBatch([pop[int(sys.argv[2]) if len(sys.argv) > 2 else 0]["program"]])
for _ in range(3):
    b.analyze(flags=2)
print("device us", b.elapsed_ms() * 1e3)
