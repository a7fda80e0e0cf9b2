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


def partition_by_direction(src_dir, world: int):
    """Per-rank source index lists (ascending) such that every direction's
    sources land on one rank and the ranks hold balanced source counts: the
    direction-sorted source list is cut into ``world`` runs of ~S/world
    sources, each cut moved to the nearest direction boundary."""
    sd = np.asarray(src_dir, dtype=np.int64)
    if world < 1:
        raise DataError("bad world size")
    order = np.argsort(sd, kind="stable")
    ds = sd[order]
    S = sd.size
    cuts = [0]
    for r in range(1, world):
        c = int(round(r * S / world))
        c = max(c, cuts[-1])
        if 0 < c < S and ds[c] == ds[c - 1]:  # snap to the nearer direction boundary
            lo = int(np.searchsorted(ds, ds[c], side="left"))
            hi = int(np.searchsorted(ds, ds[c], side="right"))
            c = lo if (c - lo) <= (hi - c) and lo >= cuts[-1] else hi
        cuts.append(min(c, S))
    cuts.append(S)
    return [np.sort(order[cuts[r]:cuts[r + 1]]) for r in range(world)]


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
