"""Host logic of the n-sharded single GEMM (SURVEY §8(f) NEXT 3,
paper_2308_15152_b200/sharded.py) on CPU: the column-block plan, and -- with
the gloo backend at world size 2/3 -- that per-rank column blocks (computed by
the oracle's emulation model standing in for the device call) gathered by the
baseline exchange reproduce the unsharded product bit for bit on every rank."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import workloads
from paper_2308_15152_b200.sharded import ShardedGemm, column_shards


def test_column_shards_cover_disjoint_balanced():
    for n in (0, 1, 7, 128, 16384, 1000):
        for world in (1, 2, 3, 4, 8):
            sh = column_shards(n, world)
            assert sh[0][0] == 0 and sh[-1][1] == n
            assert all(sh[i][1] == sh[i + 1][0] for i in range(world - 1))
            w = [b - a for a, b in sh]
            assert max(w) - min(w) <= 1
    with pytest.raises(ValueError):
        column_shards(4, 0)


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


M, N, K = 40, 30, 50


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        A, B = workloads.make_operands(1, M, N, K, seed=17)

        def local(A_, B_r, C_r):   # the oracle standing in for emu_sgemm_multicast
            if B_r.shape[0]:
                C_r.copy_(torch.from_numpy(oracle.emu_gemm("fp16", A_.numpy()[None], B_r.numpy()[None], M,
                                                           B_r.shape[0], K)[0]))

        g = ShardedGemm(M, N, K, device=torch.device("cpu"), fused=False, local=local)
        g(torch.from_numpy(A[0]), torch.from_numpy(B[0, g.n0:g.n1].copy()), "fp16")
        out.put((rank, g.C.numpy().copy(), (g.n0, g.n1), g.exchange))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_gemm_gathers_full_product(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    A, B = workloads.make_operands(1, M, N, K, seed=17)
    full = oracle.emu_gemm("fp16", A, B, M, N, K)[0]
    for rank, C, (n0, n1), exch in res:
        assert (n0, n1) == column_shards(N, world)[rank]
        assert np.array_equal(C, full), rank
        assert exch.startswith("baseline")
