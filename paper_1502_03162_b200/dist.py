"""Multi-GPU mixdown: sources partitioned across ranks, one NCCL reduce.

One process per GPU (torch.distributed, backend "nccl" on GPUs; "gloo" works
for the host-side logic tests).  Rank r renders the reflection-first partial
mix z_r of its sources; a single ``reduce(SUM)`` to the root combines the
per-ear partials (2 x (T+K-1) floats -- 23 MB at config 5) and the root
applies the resonance filter once.  No other collective is on the data path.

Partitioning by *direction* (:func:`partition_by_direction`) is what makes the
mix scale: the kernel sums the sources of a direction before its taps, so its
tap work grows with the number of distinct directions a rank holds.  A
contiguous source range of 512 of 4,096 random sources still touches ~420 of
the 1,250 directions (35% of the one-GPU tap work on 12.5% of the data); a
direction partition gives every rank ~1/N of both.
"""
from __future__ import annotations

import numpy as np

from .errors import DataError


def partition(n_src: int, world: int, rank: int):
    """Contiguous, balanced source range (s0, count) of ``rank``."""
    if world < 1 or not 0 <= rank < world:
        raise DataError("bad rank/world")
    base, extra = divmod(int(n_src), int(world))
    s0 = rank * base + min(rank, extra)
    return s0, base + (1 if rank < extra else 0)


# cost of a rank's share of the mix, in units of one source's load work: each
# source is read once; each distinct direction adds one tap pass over the
# z samples (2 ears x nnz taps), measured on B200 at ~1.6 source loads
# (cfg5: ~10 ms of loads for 4,096 sources against ~4.7 ms of taps for 1,204
# directions, DESIGN.md section 7 attribution runs)
DIRECTION_COST = 1.6


def partition_by_direction(src_dir, world: int, direction_cost: float = DIRECTION_COST):
    """Per-rank source index lists (ascending) such that every direction's
    sources land on one rank and the ranks carry balanced mix work: the
    direction-sorted source list is cut at the direction boundaries nearest
    to equal shares of (sources + direction_cost x distinct directions)."""
    sd = np.asarray(src_dir, dtype=np.int64)
    if world < 1:
        raise DataError("bad world size")
    order = np.argsort(sd, kind="stable")
    if sd.size == 0:
        return [order[:0] for _ in range(world)]
    _, starts, counts = np.unique(sd[order], return_index=True, return_counts=True)
    cum = np.cumsum(counts + float(direction_cost))  # work up to and including direction k
    total = float(cum[-1])
    bounds = [0]  # cut positions in directions
    for r in range(1, world):
        target = r * total / world
        k = int(np.searchsorted(cum, target))  # first direction whose prefix reaches the target
        # cut before k or after k, whichever lands nearer the target
        before = cum[k - 1] if k > 0 else 0.0
        k = k if (k < cum.size and abs(before - target) <= abs(cum[k] - target)) else min(k + 1, cum.size)
        bounds.append(max(k, bounds[-1]))
    bounds.append(cum.size)
    pos = np.append(starts, sd.size)  # source position of each direction boundary
    return [np.sort(order[pos[bounds[r]]:pos[bounds[r + 1]]]) for r in range(world)]


def reduce_partials(z, dst: int = 0, group=None):
    """Sum per-rank partial mixes onto ``dst`` in place (one collective)."""
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.reduce(z, dst=dst, op=dist.ReduceOp.SUM, group=group)
    return z


def sharded_mixdown(mix, y_local, s0: int, count: int, dst: int = 0, group=None, stream=None):
    """Render this rank's sources [s0, s0+count) and reduce to ``dst``.

    ``mix`` is a :class:`~paper_1502_03162_b200.batch.MixRenderer` built with the
    full source->direction map; returns the final [ears, out_len] mix on
    ``dst`` and None elsewhere.
    """
    import torch.distributed as dist

    z = mix.alloc_z()
    if count > 0:
        mix.partial(y_local, s0=s0, count=count, z=z, stream=stream)
    reduce_partials(z, dst=dst, group=group)
    rank = dist.get_rank(group) if dist.is_available() and dist.is_initialized() else 0
    if rank != dst:
        return None
    return mix.finish(z, stream=stream)
