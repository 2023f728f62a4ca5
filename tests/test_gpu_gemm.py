"""GPU parity of the emulated SGEMM (C ABI -> sm_100a tcgen05 kernels) against
the CPU oracle, element by element on the same seeded inputs.

Bars:
  * bit-exact where the method's result is exact: identity / permutation
    operands (C == reconstruct(split(B))), small-integer operands (exact
    integer product), quick returns;
  * elsewhere an element-wise bound against the "ideal" block sums
    (tests/gpu_util.py entry_bound: the tensor core's per-instruction
    truncation on the running in-block sums, and the RN steps on the running
    |C|), the in-block summation being the only freedom -- tight enough that a
    dropped correction or a doubled 2^-11 fails it at every k up to c3's 16384;
    and bit for bit against the oracle's tensor-core model (tc="sm100", fitted
    to the standalone probe, R#9);
  * north_star's accuracy gate vs FP64: rel-Frobenius <= 2x plain FP32 SGEMM
    and <= 1e-5 for k <= 4096, uniform[-1,1]; at full sizes (c2, c3) on the
    sampled outputs, with the correction-off negative control failing it.
"""
import math

import numpy as np
import pytest

import oracle
import workloads
from gpu_util import assert_bits_equal, emu_gpu, tolerance, tolerance_entries

pytestmark = pytest.mark.gpu
MODES = ["fp16", "tf32"]


def _cmp(mode, A, B, m, n, k, kblock=0, **kw):
    C = emu_gpu(mode, A, B, m, n, k, kblock=kblock, **kw)
    kb = kblock or oracle.default_kb(k)
    ref = oracle.emu_gemm(mode, A, B, m, n, k, kb=kb, alpha=kw.get("alpha", 1.0),
                          beta=kw.get("beta", 0.0), C=kw.get("C"),
                          corr=not (kw.get("flags", 0) & 1))
    tol = tolerance(mode, A, B, m, n, k, kb, corr=not (kw.get("flags", 0) & 1), alpha=kw.get("alpha", 1.0),
                    beta=kw.get("beta", 0.0), C=kw.get("C"))
    d = np.abs(C[..., :m].astype(np.float64) - ref[..., :m].astype(np.float64))
    ratio = np.max(d / np.where(tol > 0, tol, 1.0))
    assert np.all(d <= tol), f"max |gpu-oracle|/tol = {ratio:.3g}"
    # bit-exact with the oracle's measured tensor-core model (R#9)
    hw = oracle.emu_gemm(mode, A, B, m, n, k, kb=kb, alpha=kw.get("alpha", 1.0),
                         beta=kw.get("beta", 0.0), C=kw.get("C"),
                         corr=not (kw.get("flags", 0) & 1), tc="sm100")
    assert_bits_equal(C[..., :m], hw[..., :m])
    return C, ref


# ------------------------------------------------------------- exactness ----
@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("kblock", [0, 32, 128])
def test_identity_and_permutation_bit_exact(mode, kblock):
    m = n = k = 160   # two m-tiles, two n-tiles, 5 k-stages (ragged tiles)
    _, B = workloads.make_operands(1, m, n, k, seed=21)
    perm = workloads.rng(4).permutation(k)
    for P in (np.eye(k, dtype=np.float32), np.eye(k, dtype=np.float32)[perm]):
        A = workloads.colmajor(P)[None]
        C = emu_gpu(mode, A, B, m, n, k, kblock=kblock)
        ref = oracle.emu_gemm(mode, A, B, m, n, k, kb=kblock or oracle.default_kb(k))
        assert np.array_equal(C, ref)
        # B = P: C == reconstruct(split(A))
        C2 = emu_gpu(mode, B, workloads.colmajor(P)[None], m, n, k, kblock=kblock)
        ref2 = oracle.emu_gemm(mode, B, workloads.colmajor(P)[None], m, n, k, kb=kblock or oracle.default_kb(k))
        assert np.array_equal(C2, ref2)


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("shape", [(37, 29, 300, 3), (128, 128, 32, 1), (1, 1, 1, 1),
                                   (300, 260, 1000, 2), (129, 257, 33, 1)])
def test_small_integers_exact(mode, shape):
    m, n, k, batch = shape
    A, B = workloads.make_operands(batch, m, n, k, seed=8, dist="int16")
    C0 = workloads.small_int((batch, n, m), seed=9)
    exact = oracle.emu_gemm(mode, A, B, m, n, k)
    assert np.array_equal(emu_gpu(mode, A, B, m, n, k), exact)
    exact1 = oracle.emu_gemm(mode, A, B, m, n, k, beta=1.0, C=C0)
    assert np.array_equal(emu_gpu(mode, A, B, m, n, k, beta=1.0, C=C0), exact1)


# ---------------------------------------------------------------- parity ----
SHAPES = [
    (16, 64, 64, 64),        # c1 (BASELINE.json configs[0])
    (2, 200, 136, 300),      # ragged m, n, k over several tiles and k-blocks
    (1, 128, 128, 32),       # exactly one tile, one stage
    (1, 129, 257, 33),       # one past every tile edge
    (4, 256, 256, 256),      # c2 item shape
    (1, 64, 384, 1000),
    (1, 4, 4, 4096),         # long k, tiny tile
]


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: "x".join(map(str, s)))
def test_parity_uniform(mode, shape):
    batch, m, n, k = shape
    A, B = workloads.make_operands(batch, m, n, k, seed=100 + m + k)
    _cmp(mode, A, B, m, n, k)


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("kblock", [32, 64, 256, 4096])
@pytest.mark.parametrize("m", [128, 384])   # single-CTA kernel / CTA-pair TS kernel
def test_parity_kblock(mode, kblock, m):
    """every combine interval the header allows, on both kernel families; in the TS
    kernel a k-block longer than the operand ring (KB > 128) is issued in chunks"""
    n, k = 256, 1024
    A, B = workloads.make_operands(1, m, n, k, seed=77)
    _cmp(mode, A, B, m, n, k, kblock=kblock)


@pytest.mark.parametrize("mode", MODES)
def test_parity_wide_magnitudes(mode):
    m, n, k = 96, 160, 512
    A, B = workloads.make_operands(1, m, n, k, seed=78, dist="logu15")
    _cmp(mode, A, B, m, n, k)


@pytest.mark.parametrize("mode", MODES)
def test_alpha_beta(mode):
    m, n, k, batch = 150, 140, 130, 3
    A, B = workloads.make_operands(batch, m, n, k, seed=5)
    C0 = workloads.uniform((batch, n, m), seed=6)
    _cmp(mode, A, B, m, n, k, alpha=-1.5, beta=0.75, C=C0)
    # beta == 0 never reads C (NaN-filled C in emu_gpu)
    C = emu_gpu(mode, A, B, m, n, k, alpha=1.0, beta=0.0)
    assert np.all(np.isfinite(C))
    # alpha == 0 / k == 0 quick returns: C = RN(beta*C), bit-exact
    out = emu_gpu(mode, A, B, m, n, k, alpha=0.0, beta=0.5, C=C0)
    assert np.array_equal(out, (C0 * np.float32(0.5)).reshape(out.shape))
    out = emu_gpu(mode, A, B, m, n, 0, alpha=1.0, beta=0.0, C=C0)
    assert np.array_equal(out, np.zeros_like(out))


@pytest.mark.parametrize("mode", MODES)
def test_leading_dimensions_and_broadcast(mode):
    m, n, k, batch = 100, 70, 90, 3
    A, B = workloads.make_operands(batch, m, n, k, seed=12, lda=104, ldb=96)
    _cmp(mode, A, B, m, n, k)
    # strideA = 0: one A shared by all problems
    _cmp(mode, A[:1], B, m, n, k)
    _cmp(mode, A, B[:1], m, n, k)
    # ldc > m: rows between m and ldc untouched
    C0 = np.full((batch, n, m + 5), 7.0, dtype=np.float32)
    C = emu_gpu(mode, A, B, m, n, k, C=C0, ldc=m + 5)
    assert np.all(C[..., m:] == 7.0)


@pytest.mark.parametrize("mode", MODES)
def test_correction_off_policy(mode):
    """EMU_FLAG_NO_CORRECTION matches the oracle's corr=False and is
    >= 32x less accurate than the method."""
    m = n = 128
    k = 256
    A, B = workloads.make_operands(1, m, n, k, seed=41)
    Coff, _ = _cmp(mode, A, B, m, n, k, flags=1)
    Con = emu_gpu(mode, A, B, m, n, k)
    R = oracle.gemm_f64(A, B, m, n, k)
    assert oracle.rel_frobenius(Coff, R) >= 32 * oracle.rel_frobenius(Con, R)


@pytest.mark.parametrize("mode", MODES)
def test_deterministic(mode):
    m, n, k, batch = 256, 256, 512, 4
    A, B = workloads.make_operands(batch, m, n, k, seed=3)
    C1 = emu_gpu(mode, A, B, m, n, k)
    C2 = emu_gpu(mode, A, B, m, n, k)
    assert np.array_equal(C1, C2)
    # batch-sharded halves == the whole (the multi-GPU partition, R#21)
    Ch = np.concatenate([emu_gpu(mode, A[:2], B[:2], m, n, k), emu_gpu(mode, A[2:], B[2:], m, n, k)])
    assert np.array_equal(C1, Ch)


# --------------------------------------------------- A-stationary path ----
# The TS kernel keeps the split A of a whole (item, 256-row) block in TMEM when
# all of k fits its A slots (FP16 k <= 256, TF32 k <= 128), n spans >= 2 tiles of
# 128 and there are >= 148 such row blocks (api.cu dispatch).  These shapes take
# that path; with fewer row blocks the same problem takes the streaming-A path,
# which issues the same MMAs in the same order, so the two agree bit for bit.
ASTAT_SHAPES = [
    (148, 256, 256, 128),    # two row blocks per cluster, full tiles
    (150, 200, 300, 96),     # ragged m (one block), ragged n (3 tiles), 3 k-stages
    (80, 512, 384, 64),      # 2 m-pairs x 80 = 160 row blocks, 3 n-tiles
]


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("shape", ASTAT_SHAPES, ids=lambda s: "x".join(map(str, s)))
def test_astat_parity(mode, shape):
    batch, m, n, k = shape
    A, B = workloads.make_operands(batch, m, n, k, seed=300 + n + k)
    C, _ = _cmp(mode, A, B, m, n, k)
    # the streaming-A path (too few row blocks for A-stationary) gives the same bits
    half = batch // 2
    Ch = np.concatenate([emu_gpu(mode, A[:half], B[:half], m, n, k),
                         emu_gpu(mode, A[half:], B[half:], m, n, k)])
    assert np.array_equal(C, Ch)


@pytest.mark.parametrize("mode", MODES)
def test_astat_policies_and_epilogues(mode):
    batch, m, n, k = 150, 200, 300, 96
    A, B = workloads.make_operands(batch, m, n, k, seed=17)
    _cmp(mode, A, B, m, n, k, kblock=32)
    _cmp(mode, A, B, m, n, k, flags=1)
    C0 = workloads.uniform((batch, n, m), seed=18)
    _cmp(mode, A, B, m, n, k, alpha=0.5, beta=-2.0, C=C0)   # beta != 0: direct-store epilogue
    Ai, Bi = workloads.make_operands(batch, m, n, k, seed=19, dist="int16")
    assert np.array_equal(emu_gpu(mode, Ai, Bi, m, n, k), oracle.emu_gemm(mode, Ai, Bi, m, n, k))


# -------------------------------------------------------- accuracy gates ----
@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("k", [64, 256, 1024, 4096])
def test_accuracy_gate_vs_fp64(mode, k):
    """north_star: rel-Frobenius vs FP64 <= 2x plain CPU FP32 SGEMM and <= 1e-5
    (k <= 4096, uniform[-1,1]); P:557's claim of SGEMM-level accuracy."""
    m = n = 128
    for seed in (1, 2, 3):
        A, B = workloads.make_operands(1, m, n, k, seed=seed)
        R = oracle.gemm_f64(A, B, m, n, k)
        e_gpu = oracle.rel_frobenius(emu_gpu(mode, A, B, m, n, k), R)
        e_sg = oracle.rel_frobenius(oracle.sgemm_f32(A, B, m, n, k), R)
        assert e_gpu <= 2 * e_sg and e_gpu <= 1e-5, (e_gpu, e_sg)


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("k", [64, 256, 1024, 4096])
def test_accuracy_vs_cublas_sweep(mode, k):
    """P:557 ("the same accuracy as cuBLAS SGEMM") with the paper's own metric,
    max relative error, beside rel-Frobenius: batched 8 x 256 x 256 x k
    through emu_sgemm_batched and through cuBLAS FP32 (torch.bmm, TF32 off), both
    vs the FP64 oracle: rel-Frobenius within 2x of cuBLAS's; the max relative error,
    an extreme-value statistic set by near-cancelling outputs (|R| ~ 0), within 3x
    (observed up to 2.4x in TF32 mode at k <= 256, below 1x in FP16 mode)"""
    import torch
    batch, m, n = 8, 256, 256
    A, B = workloads.make_operands(batch, m, n, k, seed=700 + k)
    R = oracle.gemm_f64(A, B, m, n, k)
    old = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    try:
        Am = torch.from_numpy(A).cuda().transpose(1, 2)     # (batch, m, k)
        Bm = torch.from_numpy(B).cuda().transpose(1, 2)     # (batch, k, n)
        Cc = torch.bmm(Am, Bm).transpose(1, 2).contiguous().cpu().numpy()   # (batch, n, m) storage
    finally:
        torch.backends.cuda.matmul.allow_tf32 = old
    Ce = emu_gpu(mode, A, B, m, n, k)
    fe, fc = oracle.rel_frobenius(Ce, R), oracle.rel_frobenius(Cc, R)
    me, mc = oracle.max_rel_error(Ce, R), oracle.max_rel_error(Cc, R)
    assert fe <= 2 * fc, (fe, fc)
    assert me <= 3 * mc, (me, mc)


@pytest.mark.parametrize("mode", MODES)
def test_accuracy_vs_cublas_sgemm(mode):
    """SURVEY §8(c) pin 5: the method is as accurate as cuBLAS SGEMM on the same GPU
    (torch FP32 matmul with TF32 disabled), relative Frobenius vs FP64."""
    import torch
    m = n = 256
    k = 4096
    A, B = workloads.make_operands(1, m, n, k, seed=61)
    R = oracle.gemm_f64(A, B, m, n, k)
    old = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    try:
        Am = torch.from_numpy(A[0]).cuda().T    # column-major (k, m) storage -> m x k
        Bm = torch.from_numpy(B[0]).cuda().T    # (n, k) storage -> k x n
        Cc = (Am @ Bm).T.contiguous().cpu().numpy()[None]   # back to (n, m) storage
    finally:
        torch.backends.cuda.matmul.allow_tf32 = old
    e_cublas = oracle.rel_frobenius(Cc, R)
    e_gpu = oracle.rel_frobenius(emu_gpu(mode, A, B, m, n, k), R)
    assert e_gpu <= 2 * e_cublas, (e_gpu, e_cublas)


def test_c4_stress_range():
    """c4 (k = 4096, magnitudes 2^-30..2^30): FP16 mode overflows (R#4) and the
    range flag reports it; TF32 mode passes the accuracy gate."""
    import torch
    m = n = 256
    k = 4096
    A, B = workloads.make_operands(1, m, n, k, seed=11, dist="logu30")
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    C16 = emu_gpu("fp16", A, B, m, n, k, range_flag=flag)
    assert int(flag.item()) == 1
    assert not np.all(np.isfinite(C16))
    R = oracle.gemm_f64(A, B, m, n, k)
    C32 = emu_gpu("tf32", A, B, m, n, k)
    e_sg = oracle.rel_frobenius(oracle.sgemm_f32(A, B, m, n, k), R)
    assert oracle.rel_frobenius(C32, R) <= 2 * e_sg
    # in range (2^-30..2^15) the FP16 mode passes too, flag stays clear
    A, B = workloads.make_operands(1, m, n, k, seed=11, dist="logu15")
    flag.zero_()
    C16 = emu_gpu("fp16", A, B, m, n, k, range_flag=flag)
    assert int(flag.item()) == 0
    R = oracle.gemm_f64(A, B, m, n, k)
    assert oracle.rel_frobenius(C16, R) <= 2 * oracle.rel_frobenius(oracle.sgemm_f32(A, B, m, n, k), R)


# ---------------------------------------------- full sizes, sampled outputs ----
def _run_full(mode, batch, m, n, k, seed, flags=0):
    """the full-size problem on the GPU in the launch configuration bench.py
    times; returns the operands (host) and C (device)"""
    import torch
    import paper_2308_15152_b200 as emu
    A, B = workloads.make_operands(batch, m, n, k, seed=seed)
    dA = torch.from_numpy(A).cuda()
    dB = torch.from_numpy(B).cuda()
    dC = torch.full((batch, n, m), float("nan"), device="cuda")
    emu.emu_sgemm_batched_ex(m, n, k, 1.0, dA, m, m * k, dB, k, k * n, 0.0, dC, m, m * n, batch, mode,
                             None, None, 0, flags)
    torch.cuda.synchronize()
    return A, B, dC


def _pick(batch, m, n, seed, nsamp):
    g = workloads.rng(seed + 1)
    b = g.integers(0, batch, nsamp)
    i = g.integers(0, m, nsamp)
    j = g.integers(0, n, nsamp)
    # always include the far corners of the last problem
    b[:2], i[:2], j[:2] = batch - 1, m - 1, n - 1
    i[1], j[1] = 0, 0
    return b, i, j


def _gate(mode, A, B, m, n, k, b, i, j, got):
    """north_star's accuracy gate on the sampled outputs: rel-Frobenius vs
    FP64 <= 2x plain FP32 SGEMM (O5) on the same entries, and <= 1e-5; also the
    paper's max relative error <= 2x SGEMM's.  Returns the errors."""
    R = oracle.gemm_f64_entries(A, B, m, n, k, b, i, j)
    S = oracle.sgemm_f32_entries(A, B, m, n, k, b, i, j)
    e = (oracle.rel_frobenius(got, R), oracle.rel_frobenius(S, R),
         oracle.max_rel_error(got, R), oracle.max_rel_error(S, R))
    return e, (e[0] <= 2 * e[1] and e[0] <= 1e-5 and e[2] <= 2 * e[3])


def _sampled(mode, batch, m, n, k, seed, nsamp=384):
    import torch
    A, B, dC = _run_full(mode, batch, m, n, k, seed)
    b, i, j = _pick(batch, m, n, seed, nsamp)
    got = dC[torch.from_numpy(b), torch.from_numpy(j), torch.from_numpy(i)].cpu().numpy()
    ref = oracle.emu_gemm_entries(mode, A, B, m, n, k, b, i, j)
    tol = tolerance_entries(mode, A, B, k, b, i, j)
    d = np.abs(got.astype(np.float64) - ref)
    assert np.all(d <= tol), f"max |gpu-oracle(ideal)|/tol = {np.max(d / tol):.3g}"
    assert_bits_equal(got, oracle.emu_gemm_entries(mode, A, B, m, n, k, b, i, j, tc="sm100"))
    err, ok = _gate(mode, A, B, m, n, k, b, i, j, got)
    assert ok, f"accuracy gate failed: rel-Frobenius {err[0]:.3g} vs SGEMM {err[1]:.3g}, max-rel {err[2]:.3g} vs {err[3]:.3g}"
    return A, B


@pytest.mark.parametrize("mode", MODES)
def test_c2_full_size_sampled(mode):
    """BASELINE.json configs[1]: 1024 x 256^3 in the launch configuration
    bench.py times; 384 sampled outputs vs the oracle."""
    _sampled(mode, 1024, 256, 256, 256, seed=1)


@pytest.mark.parametrize("mode", MODES)
def test_c3_full_size_sampled(mode):
    """BASELINE.json configs[2]: one 16384^3 GEMM; sampled outputs, the
    element-wise bar, bit-exact vs the sm100 model and the accuracy gate."""
    _sampled(mode, 1, 16384, 16384, 16384, seed=7, nsamp=96)


@pytest.mark.parametrize("mode", MODES)
def test_c3_correction_off_negative_control(mode):
    """the same c3 GEMM with the correction products dropped (EMU_FLAG_NO_CORRECTION,
    P:518-519) must FAIL both the accuracy gate and the element-wise bar
    against the method's oracle: the bars discriminate at k = 16384 without
    the tensor-core model"""
    import torch
    m = n = k = 16384
    A, B, dC = _run_full(mode, 1, m, n, k, seed=7, flags=1)
    b, i, j = _pick(1, m, n, 7, 96)
    got = dC[torch.from_numpy(b), torch.from_numpy(j), torch.from_numpy(i)].cpu().numpy()
    err, ok = _gate(mode, A, B, m, n, k, b, i, j, got)
    assert not ok and err[0] > 10 * err[1], err
    ref = oracle.emu_gemm_entries(mode, A, B, m, n, k, b, i, j)          # the method (correction on)
    d = np.abs(got.astype(np.float64) - ref)
    tol = tolerance_entries(mode, A, B, k, b, i, j)
    assert np.mean(d > tol) > 0.5, np.mean(d > tol)
    # and it is what the oracle says correction-off gives, bit for bit
    assert_bits_equal(got, oracle.emu_gemm_entries(mode, A, B, m, n, k, b, i, j, corr=False, tc="sm100"))


# ----------------------------------------------------------- host entry ----
@pytest.mark.parametrize("mode", MODES)
def test_host_entry_matches_device_entry(mode):
    import paper_2308_15152_b200 as emu
    m, n, k, batch = 100, 96, 200, 5
    A, B = workloads.make_operands(batch, m, n, k, seed=9, lda=104)
    C0 = workloads.uniform((batch, n, m), seed=10)
    Ch = C0.copy()
    emu.emu_sgemm_batched_host(m, n, k, 1.25, A, 104, k * 104, B, k, n * k, 0.5, Ch, m, n * m, batch, mode)
    Cd = emu_gpu(mode, A, B, m, n, k, alpha=1.25, beta=0.5, C=C0)
    assert np.array_equal(Ch, Cd)


@pytest.mark.parametrize("mode", MODES)
def test_unaligned_operands_direct_load_path(mode):
    """lda/ldb not multiples of 4 and misaligned bases take the direct-load
    (non-TMA) path: same parity bars."""
    import torch
    import paper_2308_15152_b200 as emu
    m, n, k = 63, 61, 77
    A, B = workloads.make_operands(1, m, n, k, seed=31, lda=65, ldb=78)
    _cmp(mode, A, B, m, n, k)
    # misaligned base pointers (offset by one float) with aligned ld
    A2, B2 = workloads.make_operands(1, m, n, k, seed=32, lda=64, ldb=80)
    dA = torch.zeros(A2.size + 1, device="cuda")
    dB = torch.zeros(B2.size + 1, device="cuda")
    dA[1:] = torch.from_numpy(A2.ravel()).cuda()
    dB[1:] = torch.from_numpy(B2.ravel()).cuda()
    dC = torch.empty((n, m), device="cuda")
    emu.emu_sgemm(m, n, k, 1.0, dA.data_ptr() + 4, 64, dB.data_ptr() + 4, 80, 0.0, dC, m, mode)
    torch.cuda.synchronize()
    ref = oracle.emu_gemm(mode, A2, B2, m, n, k)[0]
    tol = tolerance(mode, A2, B2, m, n, k)[0]
    assert np.all(np.abs(dC.cpu().numpy().astype(np.float64) - ref) <= tol)
