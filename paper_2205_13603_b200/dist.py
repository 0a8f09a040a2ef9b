"""Rank helpers for one-process-per-GPU runs under torchrun.

The population is partitioned, not exchanged: every rank measures its own
slice of candidates (weak scaling), and the only cross-rank traffic is the
barrier plus the max-over-ranks reduction of the timed totals that bench.py
reports (device time is the max over ranks, never wall clock of one rank).
"""

from __future__ import annotations

import os


def rank_info():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def shard(pool_size: int, rank: int, world: int, per_rank: int):
    """Indices of this rank's slice: contiguous blocks of ``per_rank`` so the
    ranks' slices are disjoint while ``world * per_rank <= pool_size`` (and
    wrap around the pool beyond that)."""
    return [(rank * per_rank + i) % pool_size for i in range(per_rank)]


def max_over_ranks(values, device=None):
    """Element-wise max of a list of floats across ranks (no-op when not
    distributed)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(v) for v in values], dtype=torch.float64,
                     device=device if device is not None else "cpu")
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(x) for x in t.tolist()]


def sum_over_ranks(values, device=None):
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(v) for v in values], dtype=torch.float64,
                     device=device if device is not None else "cpu")
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return [float(x) for x in t.tolist()]
