"""GPU parity of the device-level API (include/emu_tcec.cuh) through its C-ABI
users: the tcec GEMM (all policies), and the structured-operand kernels
(Householder via foreach_ij, Givens via map, scan via a generated operand)
against the oracle's emulation model on the explicit operands
(oracle/structured.py).  Bit-exact where one product per output makes the
result unique (identity / permutation operands, small integers); within the
tolerance of DESIGN.md §5 otherwise."""
import math

import numpy as np
import pytest

import oracle
import workloads
from oracle import structured
from gpu_util import assert_bits_equal, tolerance, tolerance_abab

pytestmark = pytest.mark.gpu
MODES = ["fp16", "tf32"]
U = 2.0 ** -24
NO_CORR, SIMT = 1, 2


def _dev(x):
    import torch
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).cuda()


def _tcec_gemm(mode, A, B, m, n, k, flags=0, alpha=1.0, beta=0.0, C=None, kblock=0):
    import torch
    import paper_2308_15152_b200 as emu
    batch = max(A.shape[0], B.shape[0])
    lda, ldb = A.shape[2], B.shape[2]
    sA = 0 if A.shape[0] == 1 else A.shape[1] * lda
    sB = 0 if B.shape[0] == 1 else B.shape[1] * ldb
    dC = torch.full((batch, n, m), float("nan"), device="cuda") if C is None else _dev(C)
    emu.emu_tcec_gemm_batched(m, n, k, alpha, _dev(A), lda, sA, _dev(B), ldb, sB, beta, dC, m, n * m, batch,
                              mode, None, kblock, flags)
    assert emu.emu_last_launch_count() == 1
    torch.cuda.synchronize()
    return dC.cpu().numpy()


def _simt_tol(mode, A, B, m, n, k, kb=64):
    """SIMT backend: sequential FP32 FMA over each k-block (KB - 1 roundings of
    the running block sum, u each) instead of the tensor core's per-instruction
    truncation; the rest as tolerance_abab()."""
    t = tolerance_abab(mode, A, B, m, n, k) / (2 * (kb / (16 if mode == "fp16" else 8)) + 4 + 2 * math.ceil(k / kb))
    return (kb + 4 + 2 * math.ceil(k / kb)) * t


# ------------------------------------------------------------- tcec GEMM ----
@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("flags", [0, NO_CORR, SIMT, SIMT | NO_CORR])
def test_tcec_gemm_parity(mode, flags):
    """several 128 x N blocks, ragged m / n / k tails, three problems"""
    batch, m, n, k = 3, 200, 150, 200
    A, B = workloads.make_operands(batch, m, n, k, seed=61)
    C = _tcec_gemm(mode, A, B, m, n, k, flags=flags)
    ref = oracle.emu_gemm(mode, A, B, m, n, k, corr=not (flags & NO_CORR))
    tol = _simt_tol(mode, A, B, m, n, k) if flags & SIMT else \
        tolerance(mode, A, B, m, n, k, 64, corr=not (flags & NO_CORR))
    err = np.abs(C.astype(np.float64) - ref)
    assert np.all(err <= tol), np.max(err / tol)
    # bit for bit with the oracle's model of the backend (R#9 / R#26)
    assert_bits_equal(C, oracle.emu_gemm(mode, A, B, m, n, k, corr=not (flags & NO_CORR),
                                         tc="simt" if flags & SIMT else "sm100"))
    if not flags & NO_CORR:
        R = oracle.gemm_f64(A, B, m, n, k)
        assert oracle.rel_frobenius(C, R) <= 2 * oracle.rel_frobenius(oracle.sgemm_f32(A, B, m, n, k), R)


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("flags", [0, NO_CORR, SIMT])
def test_tcec_gemm_permutation_and_integers_exact(mode, flags):
    m, n, k = 130, 70, 140
    _, B = workloads.make_operands(1, m, n, k, seed=62)
    P = np.eye(k, dtype=np.float32)[workloads.rng(5).permutation(k)][:m]
    A = workloads.colmajor(P)[None]
    C = _tcec_gemm(mode, A, B, m, n, k, flags=flags)
    assert np.array_equal(C, oracle.emu_gemm(mode, A, B, m, n, k, corr=not (flags & NO_CORR)))
    Ai = workloads.small_int((1, k, m), seed=63)
    Bi = workloads.small_int((1, n, k), seed=64)
    Ci = _tcec_gemm(mode, Ai, Bi, m, n, k, flags=flags)
    exact = oracle.gemm_f64(Ai, Bi, m, n, k)
    assert np.array_equal(Ci, exact.astype(np.float32))


@pytest.mark.parametrize("mode", MODES)
def test_tcec_gemm_alpha_beta_and_kblock(mode):
    batch, m, n, k = 2, 96, 80, 256
    A, B = workloads.make_operands(batch, m, n, k, seed=65)
    C0 = workloads.uniform((batch, n, m), seed=66)
    for kb in (0, 128):
        C = _tcec_gemm(mode, A, B, m, n, k, alpha=0.5, beta=-1.5, C=C0, kblock=kb)
        ref = oracle.emu_gemm(mode, A, B, m, n, k, alpha=0.5, beta=-1.5, C=C0, kb=kb or 64)
        tol = 0.5 * tolerance_abab(mode, A, B, m, n, k, kblock=kb or 64) + 2 * U * np.abs(ref)
        assert np.all(np.abs(C.astype(np.float64) - ref) <= tol)
        assert_bits_equal(C, oracle.emu_gemm(mode, A, B, m, n, k, alpha=0.5, beta=-1.5, C=C0, kb=kb or 64,
                                             tc="sm100"))


@pytest.mark.parametrize("mode", MODES)
def test_tcec_gemm_matches_library_kernel_on_exact_cases(mode):
    """the device-API GEMM and the library's persistent kernel agree bit for bit
    wherever the result is unique (permutation operand)"""
    import paper_2308_15152_b200  # noqa: F401
    from gpu_util import emu_gpu
    m, n, k = 160, 128, 192
    _, B = workloads.make_operands(1, m, n, k, seed=67)
    A = workloads.colmajor(np.eye(k, dtype=np.float32)[workloads.rng(6).permutation(k)][:m])[None]
    assert np.array_equal(_tcec_gemm(mode, A, B, m, n, k), emu_gpu(mode, A, B, m, n, k))


# ---------------------------------------------------- structured operands ----
def _householder(mode, V, X, m, n, flags=0):
    import torch
    import paper_2308_15152_b200 as emu
    batch = V.shape[0]
    dC = torch.full((batch, n, m), float("nan"), device="cuda")
    emu.emu_tcec_householder_batched(m, n, _dev(V), m, _dev(X), m, n * m, dC, m, n * m, batch, mode, None, flags)
    torch.cuda.synchronize()
    return dC.cpu().numpy()


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("m", [16, 32, 200])
def test_householder_generated_operand(mode, m):
    """X = I: each output is one product, so C == the oracle's split-and-rebuild
    of the explicit H bit for bit (pins the in-kernel generator and its layout);
    random X: within tolerance of the oracle on the explicit H."""
    batch = 5
    V = workloads.unit_vectors(batch, m, seed=70 + m)
    I = np.broadcast_to(workloads.colmajor(np.eye(m, dtype=np.float32)), (batch, m, m))
    C = _householder(mode, V, I, m, m)
    for b in range(batch):
        Hc = workloads.colmajor(structured.householder_matrix(V[b]))[None]
        assert np.array_equal(C[b:b + 1], oracle.emu_gemm(mode, Hc, I[b:b + 1], m, m, m)), b
    n = 72
    _, X = workloads.make_operands(batch, n, n, m, seed=80 + m)
    C = _householder(mode, V, X, m, n)
    for b in range(batch):
        Hc = workloads.colmajor(structured.householder_matrix(V[b]))[None]
        ref = oracle.emu_gemm(mode, Hc, X[b:b + 1], m, n, m)
        tol = tolerance_abab(mode, Hc, X[b:b + 1], m, n, m)
        assert np.all(np.abs(C[b:b + 1].astype(np.float64) - ref) <= tol), b
        assert_bits_equal(C[b:b + 1], oracle.emu_gemm(mode, Hc, X[b:b + 1], m, n, m, tc="sm100"))


def _givens(mode, m, n, i, j, CS, X, flags=0):
    import torch
    import paper_2308_15152_b200 as emu
    batch = CS.shape[0]
    dC = torch.full((batch, n, m), float("nan"), device="cuda")
    emu.emu_tcec_givens_batched(m, n, i, j, _dev(CS), _dev(X), m, n * m, dC, m, n * m, batch, mode, None, flags)
    torch.cuda.synchronize()
    return dC.cpu().numpy()


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("mij", [(16, 2, 9), (40, 39, 0), (300, 5, 260)])
def test_givens_map_operand(mode, mij):
    m, i, j = mij
    batch = 4
    CS = workloads.rotations(batch, seed=90 + m)
    I = np.broadcast_to(workloads.colmajor(np.eye(m, dtype=np.float32)), (batch, m, m))
    C = _givens(mode, m, m, i, j, CS, I)
    for b in range(batch):
        Gc = workloads.colmajor(structured.givens_matrix(m, i, j, *CS[b]))[None]
        assert np.array_equal(C[b:b + 1], oracle.emu_gemm(mode, Gc, I[b:b + 1], m, m, m)), b
    n = 33
    _, X = workloads.make_operands(batch, n, n, m, seed=91 + m)
    C = _givens(mode, m, n, i, j, CS, X)
    for b in range(batch):
        Gc = workloads.colmajor(structured.givens_matrix(m, i, j, *CS[b]))[None]
        ref = oracle.emu_gemm(mode, Gc, X[b:b + 1], m, n, m)
        assert np.all(np.abs(C[b:b + 1].astype(np.float64) - ref) <= tolerance_abab(mode, Gc, X[b:b + 1], m, n, m))
        assert_bits_equal(C[b:b + 1], oracle.emu_gemm(mode, Gc, X[b:b + 1], m, n, m, tc="sm100"))


def _scan(mode, n, count, X, flags=0):
    import torch
    import paper_2308_15152_b200 as emu
    dY = torch.full((count, n), float("nan"), device="cuda")
    emu.emu_tcec_scan(n, count, _dev(X), n, dY, n, mode, None, flags)
    torch.cuda.synchronize()
    return dY.cpu().numpy()


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("n", [16, 100, 300])
def test_scan_generated_operand(mode, n):
    count = 70
    Xi = workloads.small_int((count, n), seed=95)
    assert np.array_equal(_scan(mode, n, count, Xi), np.cumsum(Xi.astype(np.float64), axis=1).astype(np.float32))
    X = workloads.uniform((count, n), seed=96)
    Y = _scan(mode, n, count, X)
    Lc = workloads.colmajor(structured.scan_matrix(n))[None]
    ref = oracle.emu_gemm(mode, Lc, X[None], n, count, n)[0]
    assert np.all(np.abs(Y.astype(np.float64) - ref) <= tolerance_abab(mode, Lc, X[None], n, count, n)[0])
    assert_bits_equal(Y, oracle.emu_gemm(mode, Lc, X[None], n, count, n, tc="sm100")[0])


def test_tcec_argument_errors():
    import paper_2308_15152_b200 as emu
    import torch
    x = torch.zeros(64, device="cuda")
    with pytest.raises(emu.EmuError):
        emu.emu_tcec_gemm_batched(8, 8, 8, 1.0, x, 8, 0, x, 8, 0, 0.0, x, 8, 0, 1, "fp16", None, 0, 8)
    with pytest.raises(emu.EmuError):
        emu.emu_tcec_gemm_batched(8, 8, 8, 1.0, x, 8, 0, x, 8, 0, 0.0, x, 8, 0, 1, "fp16", None, 32, 0)
    with pytest.raises(emu.EmuError):
        emu.emu_tcec_givens_batched(8, 1, 3, 3, x, x, 8, 0, x, 8, 0, 1, "fp16")


# ------------------------------------------- pipelined (warp-specialized) form ----
PIPE = 4   # EMU_FLAG_PIPELINED


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("shape", [(150, 256, 256, 256), (3, 300, 260, 320), (2, 100, 72, 2100)],
                         ids=lambda s: "x".join(map(str, s)))
def test_pipelined_gemm_is_the_library_kernel(mode, shape):
    """emu_tcec_gemm_batched with EMU_FLAG_PIPELINED runs the library's warp-specialized
    kernel through the device API's operand hooks: bit for bit the library's result
    (same kblock) and the oracle's tensor-core model, with and without correction"""
    from gpu_util import emu_gpu
    batch, m, n, k = shape
    A, B = workloads.make_operands(batch, m, n, k, seed=90 + k)
    for flags in (PIPE, PIPE | NO_CORR):
        C = _tcec_gemm(mode, A, B, m, n, k, flags=flags)
        assert np.array_equal(C, emu_gpu(mode, A, B, m, n, k, flags=flags & NO_CORR)), flags
        if batch <= 3:
            assert_bits_equal(C, oracle.emu_gemm(mode, A, B, m, n, k, corr=not (flags & NO_CORR), tc="sm100"))


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("shape", [(5, 32, 72), (160, 200, 256), (3, 256, 520)], ids=lambda s: "x".join(map(str, s)))
def test_pipelined_householder(mode, shape):
    """H generated by the library kernel's splitter warps (Ops::gen_a): the same bits
    as the synchronous tile form and as the oracle on the explicit H"""
    batch, m, n = shape
    V = workloads.unit_vectors(batch, m, seed=170 + m)
    _, X = workloads.make_operands(batch, n, n, m, seed=180 + m)
    C = _householder(mode, V, X, m, n, flags=PIPE)
    assert np.array_equal(C, _householder(mode, V, X, m, n))
    for b in sorted({0, batch - 1}):
        Hc = workloads.colmajor(structured.householder_matrix(V[b]))[None]
        assert_bits_equal(C[b:b + 1], oracle.emu_gemm(mode, Hc, X[b:b + 1], m, n, m, tc="sm100"))
        ref = oracle.emu_gemm(mode, Hc, X[b:b + 1], m, n, m)
        assert np.all(np.abs(C[b:b + 1].astype(np.float64) - ref) <= tolerance(mode, Hc, X[b:b + 1], m, n, m, 64))


def test_pipelined_rejects_simt():
    import torch
    import paper_2308_15152_b200 as emu
    x = torch.zeros(4096, device="cuda")
    with pytest.raises(emu.EmuError):
        emu.emu_tcec_gemm_batched(8, 8, 8, 1.0, x, 8, 0, x, 8, 0, 0.0, x, 8, 64, 1, "fp16", None, 0, PIPE | SIMT)
    with pytest.raises(emu.EmuError):   # no pipelined form of the map / scan users
        emu.emu_tcec_givens_batched(8, 1, 2, 3, x, x, 8, 0, x, 8, 0, 1, "fp16", None, PIPE)
