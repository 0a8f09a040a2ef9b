"""compute-sanitizer driver: one tcgen05 GEMM / bmm / conv candidate per
kernel instantiation the population reaches -- split-K mode (0: no split; 2:
arrival ticket + in-kernel zeroing + add-reduce) x epilogue (register-direct
for unsplit BN <= 32, TMA store / add-reduce for BN % 32 == 0, staged
otherwise) -- each measured a few times through the Runner (checked launch +
timed repeats), outputs compared with the fp64 reference run.  The fp32
workloads cover the 3xTF32 instantiations of the same modes.  Run as
  compute-sanitizer --tool {memcheck,racecheck,synccheck} python scripts/sanitize_tc.py
"""
import gzip
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2205_13603_b200.runner import B200Runner  # noqa: E402


def load(name):
    with gzip.open(os.path.join(ROOT, "tests", "golden", f"pop_{name}.jsonl.gz"), "rt") as fh:
        lines = fh.read().splitlines()
    return json.loads(lines[0])["e0"], [json.loads(l)["program"] for l in lines[1:2049]]


def main():
    bad = 0
    for name, fam, cfg_split, cfg_bn, dtype in (("bert_ffn", "tcgen05", 4, 3, "bf16"),
                                                ("bmm_qk", "tcgen05", 4, 3, "bf16"),
                                                ("conv2d", "tcgen05_conv", 3, 2, "bf16"),
                                                ("gmm512_tc", "tcgen05", 4, 3, "f32"),
                                                ("bmm_qk", "tcgen05", 4, 3, "f32")):
        e0, progs = load(name)
        r = B200Runner(device=0, dtype=dtype, min_repeats=2, max_repeats=2, target_ms=0.001, timeout_ms=60000.0)
        r.set_workload(e0, seed=0)
        want = r.reference_output()
        plans = r.plan_programs(progs)
        picks = {}
        for i, p in enumerate(plans):
            if p["family"] != fam or p["status"] != "OK":
                continue
            split, bn = p["cfg"][cfg_split], p["cfg"][cfg_bn]
            if fam == "tcgen05" and split == 1 and bn <= 32:
                epi = "direct"
            else:
                epi = "tma" if bn % 32 == 0 else "staged"
            picks.setdefault(("split" if split > 1 else "nosplit") + "/" + epi, i)
        for mode, i in sorted(picks.items()):
            res, = r.measure_programs([progs[i]])
            out = r.last_output().astype(np.float64)
            ok = res["status"] == "OK" and res["mismatches"] == 0 and np.array_equal(out, want)
            bad += not ok
            print(f"{name} {dtype} {fam} {mode} cfg={res['cfg']} status={res['status']} mismatches={res['mismatches']} "
                  f"exact={ok}", flush=True)
        r.close()
    print("SANITIZE_DRIVER_DONE bad=%d" % bad)


if __name__ == "__main__":
    main()
