import sys, time
sys.path.insert(0, ".")
from paper_2205_13603_b200.runner import B200Runner
from paper_2205_13603_b200.refapi import loopsched
ls = loopsched()
e0 = ls.ir.serialize(ls.gmm(512, 512, 512))
for k in range(3):
    t = time.perf_counter(); r = B200Runner(dtype="f32"); t1 = time.perf_counter()
    r.set_workload(e0); t2 = time.perf_counter()
    r.close(); t3 = time.perf_counter()
    print(f"create {1e3*(t1-t):.1f} ms  set_workload {1e3*(t2-t1):.1f} ms  close {1e3*(t3-t2):.1f} ms")
