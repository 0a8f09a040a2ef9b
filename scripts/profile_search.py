"""Where the wall time of a hardware-mode tune goes (native replay, the
look-ahead's neighbour replays and batched K7, measurement, Python search):
cProfile of plugin.tune on the GPU box, default space, 64 trials:
  python scripts/profile_search.py [gmm512|bert_ffn]"""
import cProfile
import json
import pstats
import sys
import time

sys.path.insert(0, ".")
from paper_2205_13603_b200 import plugin, replay  # noqa: E402
from paper_2205_13603_b200.refapi import loopsched  # noqa: E402

ls = loopsched()
import loopsched.costmodel  # noqa: E402,F401  (scipy import outside the timing)

which = sys.argv[1] if len(sys.argv) > 1 else "gmm512"
e0 = ls.gmm(512, 512, 512) if which == "gmm512" else ls.gmm(128, 768, 3072)
cfg = ls.SearchConfig(trials=64, batch=16, population=64, seed=0)
kw = dict(mode="hardware", device=0, dtype="f32" if which == "gmm512" else "bf16", min_repeats=3,
          max_repeats=50, target_ms=0.05, timeout_ms=5.0, timeout_factor=10.0, baseline_timeout_factor=2.0)
t0 = time.perf_counter()
ls.tune(e0, ls.default_space(), cfg)
print(json.dumps({"reference_cpu_wall_s": time.perf_counter() - t0}))
plugin.tune(e0, ls.default_space(), cfg, lookahead=False, **kw)  # warm (module loads)
for la in (False,) if which != "gmm512" else (False, True):
    nb = [0.0, 0]
    orig = replay.NativeReplayer.neighbours

    def wrapped(self, keys, _o=orig):
        t = time.perf_counter()
        r = _o(self, keys)
        nb[0] += time.perf_counter() - t
        nb[1] += r[1]["replayed"]
        return r
    replay.NativeReplayer.neighbours = wrapped
    pr = cProfile.Profile()
    t = time.perf_counter()
    pr.enable()
    plugin.tune(e0, ls.default_space(), cfg, lookahead=la, **kw)
    pr.disable()
    wall = time.perf_counter() - t
    replay.NativeReplayer.neighbours = orig
    print(json.dumps({"lookahead": la, "wall_s": wall, "neighbour_replay_s": nb[0], "neighbours": nb[1],
                      **plugin.last_tune_stats}))
    pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
