"""Multi-GPU mixdown: sources partitioned across ranks, one NCCL reduce.

One process per GPU (torch.distributed, backend "nccl" on GPUs; "gloo" works
for the host-side logic tests).  Rank r renders the reflection-first partial
mix z_r of its contiguous source range; a single ``reduce(SUM)`` to the root
combines the per-ear partials (2 x (T+K-1) floats -- 23 MB at config 5) and
the root applies the resonance filter once.  No other collective is on the
data path.
"""
from __future__ import annotations

from .errors import DataError


def partition(n_src: int, world: int, rank: int):
    """Contiguous, balanced source range (s0, count) of ``rank``."""
    if world < 1 or not 0 <= rank < world:
        raise DataError("bad rank/world")
    base, extra = divmod(int(n_src), int(world))
    s0 = rank * base + min(rank, extra)
    return s0, base + (1 if rank < extra else 0)


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
