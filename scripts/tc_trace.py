"""Per-CTA timeline of a tcgen05 candidate (globaltimer stamps), launches
chained in one CUDA graph as the runner's timed repeats:
  python scripts/tc_trace.py 49,1,64,3,3,3 16 conv2d"""
import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from conftest import load_population  # noqa: E402
from paper_2205_13603_b200 import native  # noqa: E402
from paper_2205_13603_b200.runner import B200Runner  # noqa: E402

want = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "1,1,12,64,12").split(",")]
launches = int(sys.argv[2]) if len(sys.argv) > 2 else 4
workload = sys.argv[3] if len(sys.argv) > 3 else "bert_ffn"
family = "tcgen05_conv" if workload == "conv2d" else "tcgen05"
hdr, pop = load_population(workload)
r = B200Runner(dtype="bf16")
r.set_workload(hdr["e0"])
progs = [p["program"] for p in pop]
plans = r.plan_programs(progs)
i = next(i for i, p in enumerate(plans) if p["family"] == family and p["cfg"][:len(want)] == want)
print("cfg", plans[i]["cfg"][:8])
b = progs[i].encode()
cap = 1 << 15
buf = (ctypes.c_uint64 * (8 * cap))()
n = ctypes.c_int()
native.check(native.lib().ls_runner_trace_tc(r._h, b, len(b), launches, buf, cap, ctypes.byref(n)), "trace")
a = np.frombuffer(buf, dtype=np.uint64).reshape(-1, 8)[: n.value * launches].astype(np.int64)
t0 = a[:, 0].min()
for L in range(launches):
    s = a[L * n.value:(L + 1) * n.value]
    rel = (s[:, :7] - t0) / 1000.0
    med = lambda j, i: float(np.median(rel[:, j] - rel[:, i]))
    recv = med(5, 4) if (s[:, 5] > 0).all() else float("nan")
    print(f"launch {L}: start [{rel[:,0].min():.2f},{rel[:,0].max():.2f}] setup+{med(1,0):.2f} "
          f"firstload+{med(2,1):.2f} mma_done+{med(3,2):.2f} staged+{med(4,3):.2f} "
          f"received+{recv:.2f} stored+{med(6,5) if recv == recv else med(6,4):.2f} "
          f"end [{rel[:,6].min():.2f},{rel[:,6].max():.2f}] us")
ends = [a[L * n.value:(L + 1) * n.value, 6].max() for L in range(launches)]
firsts = [a[L * n.value:(L + 1) * n.value, 2].min() for L in range(launches)]
per = np.diff(ends) / 1000.0
gap = (np.array(firsts[1:]) - np.array(ends[:-1])) / 1000.0
print(f"traced graph: {r.elapsed_ms() * 1e3 / launches:.2f} us per launch (CUDA events around the graph)")
print(f"median over launches 1..: last end -> next last end {np.median(per[1:]):.2f} us, "
      f"last end -> next first operands landed {np.median(gap[1:]):.2f} us")
