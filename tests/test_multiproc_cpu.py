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


def _check_worker(rank, world, port, out, corrupt):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        per, m, n, k = 3, 16, 12, 20

        def compute(items):
            A, B = workloads.make_operands(len(items), m, n, k, seed=7, item0=items[0])
            return torch.from_numpy(oracle.emu_gemm("fp16", A, B, m, n, k))

        lo, hi = bench.shard(rank, world, per)
        C = compute(list(range(lo, hi)))
        if corrupt and rank == 1:
            C[2, 3, 4] = float(np.nextafter(np.float32(C[2, 3, 4].item()), np.float32(np.inf)))
        rep = bench.cross_rank_check(bench.item_checksums(C), per,
                                     lambda g: bench.item_checksums(compute([g]))[0])
        if rank == 0:
            out.put(rep)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("corrupt", [False, True])
def test_cross_rank_bit_identity_check_gloo(corrupt):
    """bench.py's multi-GPU verification: gathered per-problem
    checksums against rank 0's own recomputation; a one-ulp change in one output
    of rank 1's last problem is caught"""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_check_worker, args=(r, world, port, q, corrupt)) for r in range(world)]
    for p in procs:
        p.start()
    rep = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert rep["items_checked"] == 4
    if corrupt:
        assert not rep["bit_identical"] and rep["mismatched_items"] == [5]
    else:
        assert rep["bit_identical"]


def test_item_checksums_detect_bit_changes():
    C = torch.from_numpy(workloads.uniform((2, 8, 8), seed=3))
    s0 = bench.item_checksums(C)
    D = C.clone()
    D[1, 2, 3] = float(np.nextafter(np.float32(D[1, 2, 3].item()), np.float32(0)))
    s1 = bench.item_checksums(D)
    assert s0[0] == s1[0] and s0[1] != s1[1]
    E = C.clone()
    E[0, 0, 0], E[0, 0, 1] = C[0, 0, 1], C[0, 0, 0]       # swapped elements
    assert bench.item_checksums(E)[0] != s0[0] or C[0, 0, 0] == C[0, 0, 1]
