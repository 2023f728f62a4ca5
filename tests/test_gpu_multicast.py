"""GPU checks of the fused all-gather building block:
emu_sgemm_multicast stores the same bits to every destination, its per-element
arithmetic equals emu_sgemm's (bit-identical), and an n-sharded GEMM simulated
on one GPU -- R "ranks", each multicasting its column block into all R result
buffers at its column offset -- leaves every buffer equal to the unsharded
product bit for bit.  On a multi-GPU run the destinations are peer buffers;
the kernel path is the same."""
import numpy as np
import pytest

import oracle
import workloads
from gpu_util import tolerance

pytestmark = pytest.mark.gpu
MODES = ["fp16", "tf32"]


def _t(x):
    import torch
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).cuda()


@pytest.mark.parametrize("mode", MODES)
def test_multicast_copies_equal_plain_gemm(mode):
    import torch
    import paper_2308_15152_b200 as emu
    m, n, k = 300, 260, 320
    A, B = workloads.make_operands(1, m, n, k, seed=101)
    dA, dB = _t(A[0]), _t(B[0])
    ref = torch.full((n, m), float("nan"), device="cuda")
    emu.emu_sgemm(m, n, k, 1.0, dA, m, dB, k, 0.0, ref, m, mode)
    outs = [torch.full((n, m), float("nan"), device="cuda") for _ in range(3)]
    emu.emu_sgemm_multicast(m, n, k, 1.0, dA, m, dB, k, outs, m, mode)
    assert emu.emu_last_launch_count() == 1
    torch.cuda.synchronize()
    for o in outs:
        assert torch.equal(o, ref)
    C = outs[0].cpu().numpy()[None]
    assert np.all(np.abs(C - oracle.emu_gemm(mode, A, B, m, n, k)) <= tolerance(mode, A, B, m, n, k))


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("ranks", [2, 3, 4])
def test_simulated_sharded_gemm_all_gather(mode, ranks):
    import torch
    import paper_2308_15152_b200 as emu
    from paper_2308_15152_b200.sharded import column_shards
    m, n, k = 384, 520, 256
    A, B = workloads.make_operands(1, m, n, k, seed=102)
    dA, dB = _t(A[0]), _t(B[0])
    full = torch.empty((n, m), device="cuda")
    emu.emu_sgemm(m, n, k, 1.0, dA, m, dB, k, 0.0, full, m, mode)
    Cs = [torch.full((n, m), float("nan"), device="cuda") for _ in range(ranks)]
    for n0, n1 in column_shards(n, ranks):           # "rank" r: its block into every buffer
        dsts = [c.data_ptr() + 4 * n0 * m for c in Cs]
        emu.emu_sgemm_multicast(m, n1 - n0, k, 1.0, dA, m, dB[n0:n1], k, dsts, m, mode)
    torch.cuda.synchronize()
    for c in Cs:
        assert torch.equal(c, full)


def test_sharded_gemm_single_rank():
    import torch
    import paper_2308_15152_b200 as emu
    from paper_2308_15152_b200.sharded import ShardedGemm
    m, n, k = 256, 256, 128
    A, B = workloads.make_operands(1, m, n, k, seed=103)
    g = ShardedGemm(m, n, k)
    g(_t(A[0]), _t(B[0]), "fp16")
    ref = torch.empty((n, m), device="cuda")
    emu.emu_sgemm(m, n, k, 1.0, _t(A[0]), m, _t(B[0]), k, 0.0, ref, m, "fp16")
    torch.cuda.synchronize()
    assert torch.equal(g.C, ref) and g.exchange.startswith("none")


def test_multicast_errors():
    import torch
    import paper_2308_15152_b200 as emu
    x = torch.zeros(4096, device="cuda")
    with pytest.raises(emu.EmuError):
        emu.emu_sgemm_multicast(8, 8, 8, 1.0, x, 8, x, 8, [x] * 9, 8, "fp16")
    with pytest.raises(emu.EmuError):
        emu.emu_sgemm_multicast(8, 8, 8, 1.0, x, 8, x, 8, [x, 0], 8, "fp16")
    with pytest.raises(emu.EmuError):   # lda not a multiple of 4: outside the TMA domain
        emu.emu_sgemm_multicast(6, 8, 8, 1.0, x, 6, x, 8, [x], 6, "fp16")


def test_sharded_gemm_symmetric_memory_path_one_rank():
    """the fused path's plumbing (symmetric-memory buffer, rendezvous, peer
    pointers, device barrier) on a one-rank NCCL group"""
    import socket

    import torch
    import torch.distributed as dist
    import paper_2308_15152_b200 as emu
    from paper_2308_15152_b200.sharded import ShardedGemm
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        m, n, k = 256, 384, 192
        A, B = workloads.make_operands(1, m, n, k, seed=104)
        g = ShardedGemm(m, n, k, fused=True)
        assert g.exchange.startswith("fused")
        g(_t(A[0]), _t(B[0]), "tf32")
        ref = torch.empty((n, m), device="cuda")
        emu.emu_sgemm(m, n, k, 1.0, _t(A[0]), m, _t(B[0]), k, 0.0, ref, m, "tf32")
        torch.cuda.synchronize()
        assert torch.equal(g.C, ref)
    finally:
        dist.destroy_process_group()
