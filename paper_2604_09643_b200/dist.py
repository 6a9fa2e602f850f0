"""Frame sharding across ranks and the one cross-rank exchange.

Frames are independent views (R14): forward, residual and pose gradient of frame f depend
only on p0 and (R_f, t_f).  Each rank owns a subset of frames; p0 and its Adam state are
replicated; the only collective on the data path is the SUM all-reduce of dL/dp0 (and of the
scalar loss) that pa_step requests through its callback (Stage 5 "coherently combining",
P:118).  Everything here is host plumbing; the compute runs in libpa.
"""
from __future__ import annotations

import numpy as np


def shard_frames(F: int, world: int, rank: int, cost=None) -> np.ndarray:
    """Frame indices owned by `rank`.  With per-frame costs (exact in-window counts), greedy
    longest-processing-time assignment, each rank's list sorted; else contiguous balanced blocks."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    if cost is None:
        base, extra = divmod(F, world)
        start = rank * base + min(rank, extra)
        n = base + (1 if rank < extra else 0)
        return np.arange(start, start + n, dtype=np.int64)
    cost = np.asarray(cost, dtype=np.float64)
    order = np.argsort(-cost, kind="stable")
    load = np.zeros(world)
    owner = np.empty(F, dtype=np.int64)
    for f in order:
        r = int(np.argmin(load))
        owner[f] = r
        load[r] += cost[f]
    return np.nonzero(owner == rank)[0].astype(np.int64)


def make_allreduce(group=None):
    """Return fn(tensor) that SUM-all-reduces a tensor in place over `group` (NCCL over NVLink on
    GPUs, gloo in the CPU tests)."""
    import torch.distributed as dist

    def _ar(t):
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)

    return _ar
