"""Multi-process (world_size 2, gloo on CPU) coverage of the mixdown's
host-side exchange: each rank reduces its partial mix onto rank 0 with one
collective, exactly as dist.sharded_mixdown does with NCCL on GPUs."""
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, S, T, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1502_03162_b200 import dist as tdist
    s0, n = tdist.partition(S, world, rank)
    rng = np.random.default_rng(0)
    contrib = rng.standard_normal((S, 2, T)).astype(np.float32)  # stand-in per-source partials
    z = torch.from_numpy(contrib[s0:s0 + n].sum(axis=0))
    tdist.reduce_partials(z, dst=0)
    if rank == 0:
        q.put(z.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_reduce_partials_two_ranks():
    S, T, world = 13, 257, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, S, T, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    want = np.random.default_rng(0).standard_normal((S, 2, T)).astype(np.float32).sum(axis=0)
    np.testing.assert_allclose(got, want, rtol=1e-5, atol=1e-5)
