"""Sharded measurement: round-robin dealing, in-order reassembly, one worker
process per device; rank slices and max-over-ranks with gloo (world 2)."""
import os

import pytest
import torch.multiprocessing as tmp

from fake_runner import fake_factory
from paper_2205_13603_b200 import dist, multigpu


def test_deal_covers_each_index_once():
    for n in (0, 1, 7, 64):
        for w in (1, 2, 3, 8):
            sl = multigpu.deal(n, w)
            flat = sorted(i for s in sl for i in s)
            assert flat == list(range(n))
            assert max(len(s) for s in sl) - min(len(s) for s in sl) <= 1


def test_sharded_runner_reassembles_in_order():
    texts = [f'{{"buffers": [], "root": [], "i": {i}}}' for i in range(23)]
    one = multigpu.ShardedRunner([0], factory=fake_factory)
    three = multigpu.ShardedRunner([0, 1, 2], factory=fake_factory)
    try:
        a = one.measure_programs(texts)
        b = three.measure_programs(texts)
        assert [r["latency_ns"] for r in a] == [r["latency_ns"] for r in b]
        lat = three.measure([type("C", (), {"program": t})() for t in texts])
        assert len(lat) == 23 and all(x > 0 for x in lat)
    finally:
        one.close()
        three.close()


def test_worker_error_drains_every_reply():
    # one worker fails: every reply is read before raising, so the next call
    # gets fresh answers (no stale reply left in a pipe)
    texts = [f"prog-{i}" for i in range(8)]
    sh = multigpu.ShardedRunner([0, 1], factory=fake_factory, fail_on="prog-3")
    try:
        with pytest.raises(RuntimeError, match="injected failure"):
            sh.measure_programs(texts)
        good = [f"ok-{i}" for i in range(6)]
        got = sh.measure_programs(good)
        assert [r["latency_ns"] for r in got] == [fake_factory(0)._result(t)["latency_ns"] for t in good]
        # baseline() with the loaded e0 does not re-upload (custom inputs stay)
        sh.set_workload('{"e0": 1}')
        sh.baseline('{"e0": 1}')
        assert sh.measure_programs(["x"])[0]["workloads"] == 1
        sh.baseline('{"e0": 2}')
        assert sh.measure_programs(["x"])[0]["workloads"] == 2
    finally:
        sh.close()


def test_rank_slices_are_disjoint():
    per = 100
    seen = set()
    for r in range(8):
        s = dist.shard(8192, r, 8, per)
        assert len(s) == per and not (seen & set(s))
        seen |= set(s)


def _gloo_worker(rank, world, port, q):
    import torch.distributed as d
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    d.init_process_group("gloo", rank=rank, world_size=world)
    idx = dist.shard(50, rank, world, 20)
    mx = dist.max_over_ranks([rank * 10.0 + 1.0, -rank])
    tot = dist.sum_over_ranks([len(idx)])
    q.put((rank, idx, mx, tot))
    d.barrier()
    d.destroy_process_group()


def test_gloo_world2_max_over_ranks():
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, i0, m0, t0), (r1, i1, m1, t1) = out
    assert not set(i0) & set(i1)
    assert m0 == m1 == [11.0, 0.0]
    assert t0 == t1 == [40.0]
