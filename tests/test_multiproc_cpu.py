"""Multi-process host logic of the batch-sharded path (R#21), on CPU with the
gloo backend and world size 2: each rank's shard of the global batch, the
per-problem input generation, the max-over-ranks timing reduction, and that
the sharded computation (oracle emulation model per rank, gathered) equals the
unsharded one bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import bench
import oracle
import workloads


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        per = 3
        m = n = 24
        k = 40
        lo, hi = bench.shard(rank, world, per)
        A, B = workloads.make_operands(per, m, n, k, seed=5, item0=lo)
        C = oracle.emu_gemm("fp16", A, B, m, n, k)
        gathered = [torch.zeros(per, n, m) for _ in range(world)]
        dist.all_gather(gathered, torch.from_numpy(C))
        t = bench.max_over_ranks(1.0 + rank)
        if rank == 0:
            out.put((np.concatenate([g.numpy() for g in gathered]), t, (lo, hi)))
    finally:
        dist.destroy_process_group()


def test_sharded_equals_unsharded_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    C_sharded, tmax, rng0 = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert rng0 == (0, 3)
    assert tmax == 2.0                       # max over ranks
    A, B = workloads.make_operands(6, 24, 24, 40, seed=5)
    C_full = oracle.emu_gemm("fp16", A, B, 24, 24, 40)
    assert np.array_equal(C_sharded, C_full)


def test_shard_ranges_tile_the_batch():
    for world in (1, 2, 4, 8):
        ranges = [bench.shard(r, world, 1024) for r in range(world)]
        assert ranges[0][0] == 0 and ranges[-1][1] == 1024 * world
        assert all(ranges[i][1] == ranges[i + 1][0] for i in range(world - 1))


def test_max_over_ranks_without_process_group():
    assert bench.max_over_ranks(3.5) == 3.5
