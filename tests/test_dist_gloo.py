"""Multi-process (world_size 2, gloo on CPU) coverage of the sharded mixdown's
host-side chain: direction partition -> per-rank partial mix -> one reduce
onto rank 0 -> f on the root, exactly as ``dist.MixShard`` runs it with NCCL
on GPUs.  The per-rank renderer is a host stand-in with MixRenderer's
``alloc_z`` / ``partial`` / ``finish`` methods (numpy convolutions); the
result on rank 0 is compared with the fp64 oracle's mixdown of all sources
(sum_s Renderer_e.render(y_s, dir(s)), pkg/src/toepnmf/engine/__init__.py:238-260)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from conftest import rel_l2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class HostMix:
    """CPU stand-in for batch.MixRenderer (test only): z[e] = sum_s y_s * g_{e,dir(s)}, out[e] = f_e * z[e]."""

    def __init__(self, models, src_dir, T):
        self.models = models
        self.src_dir = np.asarray(src_dir)
        self.T = T
        self.K = models[0].reflection_length
        self.ears = len(models)

    def alloc_z(self):
        return torch.zeros((self.ears, self.T + self.K - 1), dtype=torch.float64)

    def partial(self, y, z=None, **_):
        z = self.alloc_z() if z is None else z
        y = np.asarray(y, dtype=np.float64)
        acc = np.zeros((self.ears, self.T + self.K - 1))
        for i, d in enumerate(self.src_dir):
            for e, m in enumerate(self.models):
                acc[e] += np.convolve(y[i], m.reflection(int(d)))
        z.copy_(torch.from_numpy(acc))
        return z

    def finish(self, z, out=None, **_):
        zz = z.numpy()
        return torch.from_numpy(np.stack([np.convolve(m.resonance_taps, zz[e]) for e, m in enumerate(self.models)]))


def _problem(S, T, skew):
    from paper_1502_03162_b200 import synth
    cfg = synth.Config("g", ny=T, M=40, K=20, nnz=5, dirs=30, ears=2, sources=S)
    ms = synth.models(cfg, seed=3)
    sd = synth.source_directions(S, cfg.dirs, seed=4)
    if skew:
        sd[: (3 * S) // 4] = 7  # three quarters of the sources at one direction
    y = np.random.default_rng(11).standard_normal((S, T)).astype(np.float32).astype(np.float64)
    return ms, sd, y


def _worker(rank, world, port, S, T, skew, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1502_03162_b200 import dist as tdist
    ms, sd, y = _problem(S, T, skew)
    shard = tdist.MixShard(ms, sd, T, mixer=HostMix)  # world / rank from the process group
    out = shard.render(y[shard.sources])
    q.put((rank, shard.sources.tolist(), None if out is None else out.numpy()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("skew", [False, True])
def test_sharded_mixdown_two_ranks(skew):
    S, T, world = 23, 300, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, S, T, skew, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=180)
        assert p.exitcode == 0
    res.sort()
    # every source lands on exactly one rank
    allsrc = sorted(s for _, src, _ in res for s in src)
    assert allsrc == list(range(S))
    assert all(len(src) > 0 for _, src, _ in res)
    assert res[1][2] is None  # only the root holds the mix
    got = res[0][2]
    ms, sd, y = _problem(S, T, skew)
    f = np.stack([m.resonance_taps for m in ms])
    from paper_1502_03162_b200.batch import model_rows
    M = ms[0].num_taps
    want = oracle.mix_window(y, sd, f, model_rows(ms), ms[0].reflection_length, ms[0].num_directions, 0, T + M - 1)
    assert got.shape == want.shape
    for e in range(2):
        assert rel_l2(got[e], want[e]) < 1e-12
