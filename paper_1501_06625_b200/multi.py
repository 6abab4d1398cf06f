"""Batch of independent paths over several GPUs (BASELINE config 5).

Paths are independent, so the batch is split into contiguous
shards, one per rank (one process per GPU), with no collective on the data
path: each rank uploads its starts, tracks them with its own plan
(pt_track_batch) and the host gathers end points and statistics.  The only
collective is the final gather (torch.distributed, NCCL on GPUs / gloo on
CPU) -- a single path never shards ("replicas only").
"""
from __future__ import annotations

from typing import Callable, List, Optional, Tuple

import numpy as np


def shard_range(n_paths: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous shard [lo, hi) of rank `rank`; sizes differ by at most one."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    return rank * n_paths // world, (rank + 1) * n_paths // world


def step_slice(n_paths: int, per_rank: int, step: int, rank: int, world: int) -> Tuple[int, int]:
    """Weak-scaling bench slices (bench.py): at step s rank r tracks the
    contiguous paths [lo, lo + per_rank) of the batch with
    lo = ((s * world + r) * per_rank) mod n_paths, so every rank owns a fixed
    amount of work per step and N ranks together cover N slices; per_rank
    must divide n_paths (slices never wrap)."""
    if per_rank < 1 or n_paths % per_rank:
        raise ValueError("per_rank must divide n_paths")
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    lo = ((step * world + rank) * per_rank) % n_paths
    return lo, lo + per_rank


def track_batch_sharded(track: Callable[[np.ndarray], Tuple[np.ndarray, List]], starts: np.ndarray,
                        rank: int, world: int, group=None) -> Optional[Tuple[np.ndarray, np.ndarray]]:
    """Track this rank's shard with `track(starts_shard) -> (ends, stats)` and
    gather (ends, stats-as-rows) on rank 0 in path order.  stats rows are
    [status, failure_kind, steps, accepted, newton_iters, start_iters, solves].
    Returns the full arrays on rank 0, None elsewhere."""
    import torch
    import torch.distributed as dist

    lo, hi = shard_range(starts.shape[0], rank, world)
    ends, stats = track(starts[lo:hi])
    rows = np.array([[s.status, s.failure_kind, s.steps, s.accepted, s.newton_iters, s.start_iters,
                      getattr(s, "solves", 0)] for s in stats], dtype=np.int64).reshape(-1, 7)
    if world == 1:
        return ends, rows
    payload = (lo, np.ascontiguousarray(ends), rows)
    gathered = [None] * world if rank == 0 else None
    dist.gather_object(payload, gathered, dst=0, group=group)
    if rank != 0:
        return None
    gathered.sort(key=lambda x: x[0])
    return np.concatenate([g[1] for g in gathered]), np.concatenate([g[2] for g in gathered])
