"""Multi-GPU mixdown: sources partitioned across ranks, one NCCL reduce.

One process per GPU (torch.distributed, backend "nccl" on GPUs; "gloo" works
for the host-side logic tests).  Rank r renders the reflection-first partial
mix z_r of its sources; a single ``reduce(SUM)`` to the root combines the
per-ear partials (2 x (T+K-1) floats -- 23 MB at config 5) and the root
applies the resonance filter once.  No other collective is on the data path.

Reference composition being sharded: ``sum_s Renderer(model_e).render(y_s,
dir(s))`` (pkg/src/toepnmf/engine/__init__.py:238-260), reordered g-first by
the associativity the paper relies on (PAPER.md:64-71,
pkg/tests/test_acceptance.py:283-300) and split over sources by linearity.

Partitioning by *direction* (:func:`partition_by_direction`) is what makes the
mix scale: the kernel sums the sources of a direction before its taps, so its
tap work grows with the number of distinct directions a rank holds.  A
contiguous source range of 512 of 4,096 random sources still touches ~420 of
the 1,250 directions (35% of the one-GPU tap work on 12.5% of the data); a
direction partition gives every rank ~1/N of both.  A direction holding more
than a rank's share of the work is split across ranks (each rank then pays
that direction's tap pass once, on its part of the sources).

Usage (one process per GPU)::

    shard = MixShard(models, src_dir, T)          # world / rank from torch.distributed
    y = load_rows(shard.sources)                  # [len(shard.sources), T] on this GPU
    out = shard.render(y)                         # [ears, T+M-1] on the root, None elsewhere
"""
from __future__ import annotations

import numpy as np

from .errors import DataError


def partition(n_src: int, world: int, rank: int):
    """Contiguous, balanced source range (s0, count) of ``rank`` (kept for
    callers that shard by position; the mixdown uses :func:`partition_by_direction`)."""
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


def partition_cost(src_dir, idx, direction_cost: float = DIRECTION_COST) -> float:
    """Modelled mix work of a source subset: sources + direction_cost x distinct directions."""
    sd = np.asarray(src_dir, dtype=np.int64)[np.asarray(idx, dtype=np.int64)]
    return float(sd.size + direction_cost * np.unique(sd).size)


def partition_by_direction(src_dir, world: int, direction_cost: float = DIRECTION_COST, split: bool = True):
    """Per-rank source index lists (ascending, disjoint, covering every source).

    The direction-sorted source list is cut into ``world`` runs of ~equal
    modelled work (sources + direction_cost x distinct directions).  A cut is
    snapped to the nearest direction boundary -- so the direction's sources
    stay on one rank and its tap pass runs once -- unless snapping would move
    the cut by more than 2% of a rank's share (and more than a direction's
    own cost) from its target; then (with ``split``) the cut falls inside the
    direction and both ranks run its tap pass on their part of its sources.
    Deterministic in ``src_dir``."""
    sd = np.asarray(src_dir, dtype=np.int64)
    world = int(world)
    if world < 1:
        raise DataError("bad world size")
    if sd.ndim != 1:
        raise DataError("src_dir must be 1-d")
    order = np.argsort(sd, kind="stable")
    S = sd.size
    if S == 0:
        return [order[:0] for _ in range(world)]
    ss = sd[order]
    new_dir = np.ones(S, dtype=bool)
    new_dir[1:] = ss[1:] != ss[:-1]
    # cum[i] = work of the sorted prefix [0, i): i sources + dc x directions started before i
    cum = np.concatenate([[0.0], np.arange(1, S + 1) + direction_cost * np.cumsum(new_dir)])
    starts = np.flatnonzero(new_dir)  # direction boundaries (positions where a direction begins)
    bounds = np.append(starts, S)
    total = float(cum[-1])
    cuts = [0]
    for r in range(1, world):
        target = r * total / world
        # nearest direction boundary
        k = int(np.searchsorted(cum[bounds], target))
        cands = [bounds[j] for j in (k - 1, k) if 0 <= j < bounds.size]
        b = min(cands, key=lambda p: (abs(cum[p] - target), p))
        cut = int(b)
        if split and abs(cum[b] - target) > max(direction_cost + 1.0, 0.02 * total / world):
            # inside a direction: the first position whose prefix work reaches the target
            cut = int(min(S, np.searchsorted(cum, target)))
        cuts.append(max(cut, cuts[-1]))
    cuts.append(S)
    return [np.sort(order[cuts[r]:cuts[r + 1]]) for r in range(world)]


def reduce_partials(z, dst: int = 0, group=None):
    """Sum per-rank partial mixes onto ``dst`` in place (one collective)."""
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.reduce(z, dst=dst, op=dist.ReduceOp.SUM, group=group)
    return z


def _world_rank(world, rank, group):
    if world is not None and rank is not None:
        return int(world), int(rank)
    try:
        import torch.distributed as dist
        if dist.is_available() and dist.is_initialized():
            return dist.get_world_size(group), dist.get_rank(group)
    except ImportError:
        pass
    return 1, 0


class MixShard:
    """This rank's share of a sharded mixdown over ``world`` ranks.

    ``sources`` are the global source indices (ascending) the rank must hold,
    chosen by :func:`partition_by_direction`; :meth:`render` takes them as the
    rows of a [len(sources), T] array, renders their reflection-first partial
    mix, reduces it onto ``dst`` with one collective and applies f there.
    ``mixer`` builds the per-rank renderer (default
    :class:`~paper_1502_03162_b200.batch.MixRenderer`; the multi-process CPU
    tests substitute a host stand-in with the same ``alloc_z`` / ``partial`` /
    ``finish`` methods)."""

    def __init__(self, models, src_dir, T: int, world: int | None = None, rank: int | None = None, group=None,
                 mixer=None, direction_cost: float = DIRECTION_COST):
        if mixer is None:
            from .batch import MixRenderer as mixer
        self.world, self.rank = _world_rank(world, rank, group)
        if not 0 <= self.rank < self.world:
            raise DataError("bad rank/world")
        self.group = group
        self.src_dir = np.ascontiguousarray(src_dir, dtype=np.int32)
        if self.src_dir.ndim != 1 or self.src_dir.size == 0:
            raise DataError("need at least one source")
        self.parts = partition_by_direction(self.src_dir, self.world, direction_cost)
        self.sources = self.parts[self.rank]
        self.T = int(T)
        # a rank without sources still contributes zeros to the reduce (and the
        # root still applies f): its renderer holds one placeholder source
        self.empty = self.sources.size == 0
        sd_local = self.src_dir[self.sources] if not self.empty else self.src_dir[:1]
        self.mix = mixer(models, sd_local, self.T)

    def alloc_z(self):
        return self.mix.alloc_z()

    def partial(self, y_local, z=None, stream=None, check_finite: bool = True):
        """This rank's partial z (zeros for an empty shard); no collective."""
        if z is None:
            z = self.mix.alloc_z()
        if self.empty:
            z.zero_()
            return z
        if y_local.shape[0] != self.sources.size:
            raise DataError("expected %d source rows, got %d" % (self.sources.size, y_local.shape[0]))
        return self.mix.partial(y_local, z=z, stream=stream, check_finite=check_finite)

    def render(self, y_local, dst: int = 0, z=None, out=None, stream=None, check_finite: bool = True):
        """Partial mix -> one reduce onto ``dst`` -> f on ``dst``.  Returns the
        [ears, T+M-1] mix on ``dst`` and None on the other ranks."""
        z = self.partial(y_local, z=z, stream=stream, check_finite=check_finite)
        reduce_partials(z, dst=dst, group=self.group)
        if self.rank != dst:
            return None
        return self.mix.finish(z, out=out, stream=stream)


def sharded_mixdown(models, src_dir, T: int, y_local, world: int | None = None, rank: int | None = None,
                    dst: int = 0, group=None, stream=None):
    """One-shot :class:`MixShard` render; ``y_local`` holds the rows
    ``MixShard(...).sources`` (see :func:`partition_by_direction`)."""
    return MixShard(models, src_dir, T, world, rank, group).render(y_local, dst=dst, stream=stream)
