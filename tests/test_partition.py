"""Direction partition of the sharded mixdown (dist.partition_by_direction): coverage,
balance of the modelled work, and splitting of directions heavier than a rank's share."""
import numpy as np
import pytest

from paper_1502_03162_b200 import dist as tdist
from paper_1502_03162_b200 import synth


def _check_cover(parts, S):
    allsrc = np.sort(np.concatenate(parts))
    assert np.array_equal(allsrc, np.arange(S))
    for p in parts:
        assert np.all(np.diff(p) > 0)  # ascending, no duplicates


def _costs(sd, parts):
    return np.array([tdist.partition_cost(sd, p) for p in parts])


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_cfg5_uniform_directions(world):
    cfg = synth.CONFIGS["cfg5"]
    sd = synth.source_directions(cfg.sources, cfg.dirs, seed=5)
    parts = tdist.partition_by_direction(sd, world)
    assert len(parts) == world
    _check_cover(parts, cfg.sources)
    c = _costs(sd, parts)
    assert c.max() / c.mean() < 1.01
    # at most world-1 directions are split (each cut touches at most one)
    owners = {}
    for r, p in enumerate(parts):
        for d in np.unique(sd[p]):
            owners.setdefault(int(d), set()).add(r)
    assert sum(len(v) > 1 for v in owners.values()) <= world - 1
    # the direction partition holds ~1/world of the distinct directions per rank
    nd = np.unique(sd).size
    for p in parts:
        assert np.unique(sd[p]).size <= 1.05 * nd / world + 2


@pytest.mark.parametrize("world", [2, 4, 8])
def test_single_heavy_direction_is_split(world):
    S = 4096
    sd = np.zeros(S, dtype=np.int32)
    parts = tdist.partition_by_direction(sd, world)
    _check_cover(parts, S)
    sizes = np.array([p.size for p in parts])
    assert sizes.max() - sizes.min() <= 2
    # without splitting one rank would hold everything
    unsplit = tdist.partition_by_direction(sd, world, split=False)
    assert max(p.size for p in unsplit) == S


def test_zipf_skew_balanced():
    rng = np.random.default_rng(0)
    S, D = 4096, 1250
    w = 1.0 / np.arange(1, D + 1) ** 1.2
    sd = rng.choice(D, size=S, p=w / w.sum()).astype(np.int32)
    for world in (2, 4, 8):
        parts = tdist.partition_by_direction(sd, world)
        _check_cover(parts, S)
        c = _costs(sd, parts)
        assert c.max() / c.mean() < 1.05, (world, c)


def test_more_ranks_than_sources():
    sd = np.array([3, 1, 3], dtype=np.int32)
    parts = tdist.partition_by_direction(sd, 8)
    _check_cover(parts, 3)
    assert sum(p.size == 0 for p in parts) >= 5


def test_mixshard_rows_and_empty_rank():
    """MixShard picks the rank's rows; an empty rank contributes zeros (host stand-in renderer)."""
    import torch

    class Stub:
        def __init__(self, models, src_dir, T):
            self.src_dir = np.asarray(src_dir)

        def alloc_z(self):
            return torch.ones((2, 8))

        def partial(self, y, z=None, **_):
            z.fill_(float(y.sum()))
            return z

        def finish(self, z, out=None, **_):
            return z

    sd = np.array([0, 0, 5], dtype=np.int32)
    shards = [tdist.MixShard([None], sd, 4, world=4, rank=r, mixer=Stub) for r in range(4)]
    assert sorted(int(s) for sh in shards for s in sh.sources) == [0, 1, 2]
    empty = [sh for sh in shards if sh.empty]
    assert empty
    z = empty[0].partial(np.zeros((0, 4)))
    assert float(z.abs().sum()) == 0.0
    full = [sh for sh in shards if not sh.empty][0]
    with pytest.raises(Exception):
        full.partial(np.zeros((full.sources.size + 1, 4)))
