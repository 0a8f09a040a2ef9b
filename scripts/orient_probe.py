"""Operand-orientation probe for the BERT-FFN contraction: the tcgen05 family's
per-configuration best latency at gmm(128,768,3072) (tokens on the UMMA M side,
the product orientation) next to gmm(768,128,3072) (the same bytes with the 768
output features on UMMA M and the 128 tokens on UMMA N -- the swapped
orientation, output stored [feature][token]).  Same box, same process:
  python scripts/orient_probe.py [samples]"""
import os
import random
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2205_13603_b200.refapi import loopsched  # noqa: E402
from paper_2205_13603_b200 import tensor_core as T  # noqa: E402
from paper_2205_13603_b200.runner import B200Runner  # noqa: E402

ls = loopsched()
from loopsched.spaces import run_generator  # noqa: E402

samples = int(sys.argv[1]) if len(sys.argv) > 1 else 600
gen = T.space_from_config({"modules": [{"tensor_core": {"pipeline": True}}]})
for (n, m, k) in ((128, 768, 3072), (768, 128, 3072)):
    e0 = ls.gmm(n, m, k)
    rng = random.Random(7)
    seen = {}
    for _ in range(samples):
        prog, _ = run_generator(e0, gen, rng.randrange(2 ** 62))
        seen.setdefault(ls.ir.structural_hash(prog), prog)
    texts = [ls.ir.serialize(p) for p in seen.values()]
    r = B200Runner(dtype="bf16", min_repeats=200, max_repeats=2000, target_ms=1.0, timeout_ms=5.0)
    r.set_workload(ls.ir.serialize(e0))
    plans = r.plan_programs(texts)
    best = {}
    for t, p in zip(texts, plans):
        if p["family"] != "tcgen05" or p["status"] != "OK":
            continue
        x, = r.measure_programs([t])
        key = tuple(p["cfg"][:8])
        if x["status"] == "OK" and (key not in best or x["latency_ns"] < best[key]):
            best[key] = x["latency_ns"]
    r.close()
    flops = 2.0 * n * m * k
    print(f"== gmm({n},{m},{k}): {len(texts)} programs, {len(best)} tcgen05 configurations")
    for key, ns in sorted(best.items(), key=lambda kv: kv[1])[:12]:
        print(f"  {ns / 1e3:7.2f} us {flops / ns / 1e3:7.1f} TF/s cfg {list(key)}")
