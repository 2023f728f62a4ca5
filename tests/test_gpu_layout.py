"""Row-major storage at the C ABI (emu_sgemm_batched_layout, NEXT row 2) and the
torch-facing `matmul` marshalling: against the oracle on the equivalent
column-major problem (bit-identical to the column-major entry on the swapped
problem, within the parity tolerance of the oracle), all transpose pairs."""
import numpy as np
import pytest

import oracle
import workloads
from gpu_util import tolerance

pytestmark = pytest.mark.gpu
MODES = ["fp16", "tf32"]


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("trans", ["NN", "TN", "NT", "TT"])
def test_row_major_matmul_parity(mode, trans):
    import torch
    import paper_2308_15152_b200 as emu
    batch, m, n, k = 3, 200, 136, 264
    g = workloads.rng(7)
    Am = workloads.uniform((batch, m, k), seed=111)      # math matrices (row index = i)
    Bm = workloads.uniform((batch, k, n), seed=112)
    A = torch.from_numpy(Am).cuda()
    B = torch.from_numpy(Bm).cuda()
    if trans[0] == "T":   # same math matrix, column-contiguous view
        A = torch.from_numpy(np.ascontiguousarray(np.swapaxes(Am, 1, 2))).cuda().transpose(1, 2)
    if trans[1] == "T":
        B = torch.from_numpy(np.ascontiguousarray(np.swapaxes(Bm, 1, 2))).cuda().transpose(1, 2)
    C = emu.matmul(A, B, mode).cpu().numpy()
    Ac, Bc = workloads.colmajor(Am), workloads.colmajor(Bm)
    ref = workloads.math_view(oracle.emu_gemm(mode, Ac, Bc, m, n, k), m)
    tol = workloads.math_view(tolerance(mode, Ac, Bc, m, n, k), m)
    assert np.all(np.abs(C.astype(np.float64) - ref) <= tol)
    del g


@pytest.mark.parametrize("mode", MODES)
def test_row_major_exact_and_broadcast(mode):
    import torch
    import paper_2308_15152_b200 as emu
    m, n, k = 96, 72, 160
    Ai = workloads.small_int((4, m, k), seed=113)
    Bi = workloads.small_int((k, n), seed=114)                 # 2-D: shared by the 4 problems
    C = emu.matmul(torch.from_numpy(Ai).cuda(), torch.from_numpy(Bi).cuda(), mode).cpu().numpy()
    assert np.array_equal(C, (Ai.astype(np.float64) @ Bi.astype(np.float64)).astype(np.float32))
    # row-major through the C ABI == column-major on the swapped problem, bit for bit
    Am = workloads.uniform((m, k), seed=115)
    Bm = workloads.uniform((k, n), seed=116)
    dA, dB = torch.from_numpy(Am).cuda(), torch.from_numpy(Bm).cuda()
    c_rm = torch.empty((m, n), device="cuda")
    emu.emu_sgemm_batched_layout(emu.EMU_ROW_MAJOR, "N", "N", m, n, k, 1.0, dA, k, 0, dB, n, 0, 0.0, c_rm, n, 0,
                                 1, mode)
    c_cm = torch.empty((m, n), device="cuda")   # C^T column-major = C row-major
    emu.emu_sgemm_batched(n, m, k, 1.0, dB, n, 0, dA, k, 0, 0.0, c_cm, n, 0, 1, mode)
    torch.cuda.synchronize()
    assert torch.equal(c_rm, c_cm)


def test_matmul_argument_errors():
    import torch
    import paper_2308_15152_b200 as emu
    a = torch.zeros(8, 8, device="cuda")
    with pytest.raises(ValueError):
        emu.matmul(a, torch.zeros(7, 8, device="cuda"))
    with pytest.raises(TypeError):
        emu.matmul(a.double(), a)
    with pytest.raises(emu.EmuError):
        emu.emu_sgemm_batched_layout(2, "N", "N", 8, 8, 8, 1.0, a, 8, 0, a, 8, 0, 0.0, a, 8, 0, 1, "fp16")


@pytest.mark.parametrize("mode", MODES)
def test_cuda_graph_capture_replay(mode):
    """the device entries allocate nothing and only launch on the given stream, so
    they can be captured in a CUDA graph; replays give the eager bits"""
    import torch
    import paper_2308_15152_b200 as emu
    batch, m, n, k = 16, 64, 64, 64
    A, B = workloads.make_operands(batch, m, n, k, seed=117)
    dA, dB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    eager = torch.empty((batch, n, m), device="cuda")
    emu.emu_sgemm_batched(m, n, k, 1.0, dA, m, m * k, dB, k, n * k, 0.0, eager, m, m * n, batch, mode)
    out = torch.full((batch, n, m), float("nan"), device="cuda")
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            emu.emu_sgemm_batched(m, n, k, 1.0, dA, m, m * k, dB, k, n * k, 0.0, out, m, m * n, batch, mode)
    for _ in range(3):
        out.fill_(float("nan"))
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(out, eager)
