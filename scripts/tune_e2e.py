"""End-to-end tuning on the B200 through the reference's unchanged search
(plugin.py), BASELINE configs 1 and 5:

  python scripts/tune_e2e.py gmm512      # config 1: gmm 512^3 fp32, 64 trials, seed 0
  python scripts/tune_e2e.py gmm512_tc   # config 1 with the tcgen05 module (fp32 tiles as 3xTF32)
  python scripts/tune_e2e.py bert [N]    # config 5: BERT-base tasks, N trials (default 2000)

Needs the reference package importable (baseline/_ref).  Prints one JSON
document (reference report keys + hardware section / scheduler summary)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2205_13603_b200 import plugin  # noqa: E402
from paper_2205_13603_b200.refapi import loopsched  # noqa: E402


def peak():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["bf16_tflops"]
    except Exception:
        return None


def gmm512(tc=False):
    ls = loopsched()
    e0 = ls.gmm(512, 512, 512)
    if tc:
        from paper_2205_13603_b200.tensor_core import b200_space
    space = b200_space if tc else ls.default_space
    cfg = ls.SearchConfig(trials=64, batch=16, population=64, seed=0)
    t0 = time.perf_counter()
    rep_p = plugin.tune(e0, space(), cfg, mode="parity")
    t_par = time.perf_counter() - t0
    t0 = time.perf_counter()
    bf16 = peak()
    rep, doc = plugin.tune_with_records(e0, space(), cfg, mode="hardware", dtype="f32",
                                        peak_tflops=bf16 / 6 if tc and bf16 else 148 * 128 * 2 * 1.965e9 / 1e12,
                                        peak_source="3xTF32 roof (measured bf16 / 6)" if tc and bf16
                                        else "fp32 SIMT nominal", timeout_ms=5.0, timeout_factor=10.0,
                                        min_repeats=3, max_repeats=50, target_ms=0.05)
    t_hw = time.perf_counter() - t0
    return {"config": "gmm512 fp32, %s, 64 trials, seed 0" % ("default space + use_tensor_core" if tc else "default space"),
            "parity_mode": {"best_cycles": str(rep_p.best.latency), "wall_s": t_par, "trials": len(rep_p.log)},
            "hardware_mode": {"wall_s": t_hw, "trials": len(rep.log), "best_ns": float(rep.best.latency),
                              "baseline_ns": float(rep.baseline_latency), "speedup": rep.speedup,
                              "hardware": doc["hardware"]["best"]}}


def bert(total):
    from paper_2205_13603_b200.runner import B200Runner
    from paper_2205_13603_b200.tensor_core import b200_space
    from paper_2205_13603_b200.task_scheduler import TaskScheduler, bert_tasks
    tasks = bert_tasks()
    runners = {}

    def runner_for(t):
        if t.name not in runners:
            r = B200Runner(device=0, dtype="bf16", min_repeats=3, max_repeats=50, target_ms=0.05,
                           timeout_ms=5.0, timeout_factor=10.0)
            r.set_workload(t.e0)
            runners[t.name] = r
        return runners[t.name]

    sch = TaskScheduler(tasks, total, round_trials=64, batch=16, population=64, seed=0,
                        generator_for=lambda t: b200_space(), runner_for=runner_for, mode="hardware")
    t0 = time.perf_counter()
    summary = sch.run()
    summary["wall_s"] = time.perf_counter() - t0
    summary["config"] = f"BERT-base seq 128: {len(tasks)} tasks, {total} trials, 1 B200"
    from paper_2205_13603_b200.records import contraction_flops
    summary["network_gflop"] = sum(contraction_flops(t.e0) * t.weight for t in tasks) / 1e9
    summary["network_tflops_at_best"] = summary["network_gflop"] / (summary["objective"] * 1e-9) / 1e3
    return summary


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "gmm512"
    if what.startswith("gmm512"):
        out = gmm512(tc=what == "gmm512_tc")
    else:
        out = bert(int(sys.argv[2]) if len(sys.argv) > 2 else 2000)
    print(json.dumps(out, default=str))
