"""Pins for the oracle's GEMMs against things other than themselves:
exact integer products, identity/permutation structure, exact rational
products (Python Fractions) with the componentwise error bound derived in
DESIGN.md §3, the correction-off negative control, numpy's float64 matmul,
and the paper's accuracy claim (emulated accuracy at FP32-SGEMM level).
"""
import fractions
import math

import numpy as np
import pytest

import oracle
import workloads

U = 2.0 ** -24
MODES = ["fp16", "tf32"]


def _ops(m, n, k, seed, dist="uniform", batch=1):
    return workloads.make_operands(batch, m, n, k, seed, dist)


# ------------------------------------------------------- structure pins ----
@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("kb", [16, 64, 256])
def test_identity_and_permutation_give_reconstruct(mode, kb):
    """A = I or a permutation P (one nonzero product per output) => the output
    is hi + lo*2^-11 of B's entry, rounded once: C == reconstruct(split(B))
    bit for bit (and symmetric for B = P)."""
    m = n = k = 48
    _, B = _ops(m, n, k, seed=21)
    Bm = workloads.math_view(B[0], k)
    perm = workloads.rng(4).permutation(k)
    for P in (np.eye(k, dtype=np.float32), np.eye(k, dtype=np.float32)[perm]):
        A = workloads.colmajor(P)[None]
        C = oracle.emu_gemm(mode, A, B, m, n, k, kb=kb)
        hi, lo = oracle.split_values(mode, Bm)
        expect = P @ oracle.reconstruct(mode, hi, lo).astype(np.float64)
        assert np.array_equal(workloads.math_view(C[0], m), expect.astype(np.float32))
        # B = P
        Bp = workloads.colmajor(P)[None]
        Am = workloads.math_view(B[0], k)  # reuse the random data as A
        C2 = oracle.emu_gemm(mode, workloads.colmajor(Am)[None], Bp, m, n, k, kb=kb)
        hi, lo = oracle.split_values(mode, Am)
        expect2 = oracle.reconstruct(mode, hi, lo).astype(np.float64) @ P
        assert np.array_equal(workloads.math_view(C2[0], m), expect2.astype(np.float32))


@pytest.mark.parametrize("mode", MODES)
def test_small_integers_exact(mode):
    """integer entries in [-16, 16] split exactly (lo = 0) and all partial sums
    stay below 2^24: every output equals the exact integer product, for ragged
    shapes, several k-blocks, batch strides, alpha = 1, beta in {0, 1}."""
    m, n, k, batch = 37, 29, 300, 3
    A, B = _ops(m, n, k, seed=8, dist="int16", batch=batch)
    C0 = workloads.small_int((batch, n, m), seed=9)
    Ai = np.rint(workloads.math_view(A, m)).astype(np.int64)
    Bi = np.rint(workloads.math_view(B, k)).astype(np.int64)
    exact = np.einsum("bik,bkj->bij", Ai, Bi)
    C = oracle.emu_gemm(mode, A, B, m, n, k, kb=64)
    assert np.array_equal(workloads.math_view(C, m), exact.astype(np.float32))
    C1 = oracle.emu_gemm(mode, A, B, m, n, k, beta=1.0, C=C0, kb=64)
    assert np.array_equal(workloads.math_view(C1, m),
                          (exact + workloads.math_view(C0, m).astype(np.int64)).astype(np.float32))


def _exact_product(Am, Bm):
    """exact rational A @ B (tiny sizes only)."""
    m, k = Am.shape
    n = Bm.shape[1]
    Af = [[fractions.Fraction(float(Am[i, p])) for p in range(k)] for i in range(m)]
    Bf = [[fractions.Fraction(float(Bm[p, j])) for j in range(n)] for p in range(k)]
    return np.array([[float(sum(Af[i][p] * Bf[p][j] for p in range(k))) for j in range(n)]
                     for i in range(m)], dtype=np.float64), Af, Bf


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("dist", ["uniform", "logu15"])
def test_componentwise_bound_vs_exact(mode, dist):
    """|C - AB|_ij <= (10 + ceil(k/KB)) u (|A||B|)_ij, the first-order bound of
    DESIGN.md §3 with an ideal (exact, one-rounding) block sum: 4u dropped
    lo*lo, 2u+2u lo roundings, one RN per block sum and per combine, one RN per
    cross-block add.  A dropped correction product, a wrong sign, index or a
    transposed operand all exceed it by orders of magnitude."""
    m, n, k, kb = 6, 5, 96, 32
    A, B = _ops(m, n, k, seed=31, dist=dist)
    Am = workloads.math_view(A[0], m)
    Bm = workloads.math_view(B[0], k)
    exact, _, _ = _exact_product(Am, Bm)
    C = workloads.math_view(oracle.emu_gemm(mode, A, B, m, n, k, kb=kb)[0], m).astype(np.float64)
    absAB = np.abs(Am.astype(np.float64)) @ np.abs(Bm.astype(np.float64))
    gamma = 10 + math.ceil(k / kb)
    assert np.all(np.abs(C - exact) <= gamma * U * absAB)
    # and the bound is not vacuous: correction off violates it
    Cn = workloads.math_view(oracle.emu_gemm(mode, A, B, m, n, k, kb=kb, corr=False)[0], m)
    assert np.any(np.abs(Cn.astype(np.float64) - exact) > gamma * U * absAB)


@pytest.mark.parametrize("mode", MODES)
def test_correction_off_negative_control(mode):
    """without the two correction products the error is >= 32x worse."""
    m = n = 32
    k = 256
    A, B = _ops(m, n, k, seed=41)
    R = oracle.gemm_f64(A, B, m, n, k)
    e_on = oracle.rel_frobenius(oracle.emu_gemm(mode, A, B, m, n, k), R)
    e_off = oracle.rel_frobenius(oracle.emu_gemm(mode, A, B, m, n, k, corr=False), R)
    assert e_off >= 32 * e_on


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("k", [64, 256, 1024])
def test_accuracy_claim_vs_fp32_sgemm(mode, k):
    """P:557 ("accuracy remains the same with cuBLAS SGEMM"), north_star gate:
    rel-Frobenius(emulation) <= 2 x rel-Frobenius(plain FP32 SGEMM) and <= 1e-5,
    uniform[-1,1], three seeds."""
    m = n = 32
    for seed in (1, 2, 3):
        A, B = _ops(m, n, k, seed=seed)
        R = oracle.gemm_f64(A, B, m, n, k)
        e_emu = oracle.rel_frobenius(oracle.emu_gemm(mode, A, B, m, n, k), R)
        e_sg = oracle.rel_frobenius(oracle.sgemm_f32(A, B, m, n, k), R)
        assert e_emu <= 2 * e_sg and e_emu <= 1e-5, (e_emu, e_sg)


def test_fp16_overflow_is_nonfinite_and_tf32_is_not():
    """R#4: FP16 hi overflows for |x| >= 65520 (c4's 2^30 magnitudes) and the
    output is non-finite; TF32 keeps binary32's range."""
    m = n = 8
    k = 64
    A, B = _ops(m, n, k, seed=5, dist="logu30")
    C16 = oracle.emu_gemm("fp16", A, B, m, n, k)
    assert not np.all(np.isfinite(C16))
    C32 = oracle.emu_gemm("tf32", A, B, m, n, k)
    R = oracle.gemm_f64(A, B, m, n, k)
    assert np.all(np.isfinite(C32))
    assert oracle.rel_frobenius(C32, R) <= 2 * oracle.rel_frobenius(oracle.sgemm_f32(A, B, m, n, k), R) + 1e-7


# ---------------------------------------------------- alpha/beta & BLAS ----
@pytest.mark.parametrize("mode", MODES)
def test_alpha_beta_semantics(mode):
    m, n, k = 9, 7, 33
    A, B = _ops(m, n, k, seed=2)
    C0 = workloads.uniform((1, n, m), seed=3)
    base = oracle.emu_gemm(mode, A, B, m, n, k)
    # beta == 0 never reads C (NaN garbage must not propagate, R#19)
    nanC = np.full((1, n, m), np.nan, dtype=np.float32)
    assert np.array_equal(oracle.emu_gemm(mode, A, B, m, n, k, beta=0.0, C=nanC), base)
    # alpha == 0 => C = beta*C, A and B unread (Inf in A must not propagate)
    Ainf = A.copy()
    Ainf[0, 0, 0] = np.inf
    out = oracle.emu_gemm(mode, Ainf, B, m, n, k, alpha=0.0, beta=0.5, C=C0)
    assert np.array_equal(out, (C0 * np.float32(0.5)).astype(np.float32))
    # alpha, beta general: one fma of the model's accumulator
    out = oracle.emu_gemm(mode, A, B, m, n, k, alpha=2.0, beta=-1.0, C=C0)
    expect = np.float32(2.0) * base + (np.float32(-1.0) * C0)   # 2x is exact
    assert np.array_equal(out, expect.astype(np.float32))


@pytest.mark.parametrize("mode", MODES)
def test_entries_match_full(mode):
    m, n, k, batch = 20, 24, 100, 3
    A, B = _ops(m, n, k, seed=6, batch=batch)
    C0 = workloads.uniform((batch, n, m), seed=7)
    full = oracle.emu_gemm(mode, A, B, m, n, k, alpha=1.5, beta=0.25, C=C0, kb=32)
    g = workloads.rng(9)
    b = g.integers(0, batch, 50)
    i = g.integers(0, m, 50)
    j = g.integers(0, n, 50)
    ent = oracle.emu_gemm_entries(mode, A, B, m, n, k, b, i, j, alpha=1.5, beta=0.25, C=C0, kb=32)
    assert np.array_equal(ent, full[b, j, i])


def test_strided_broadcast_batch():
    """strideA = 0 (one A shared by all items) equals explicit replication."""
    m, n, k, batch = 16, 12, 40, 4
    A, B = _ops(m, n, k, seed=12, batch=batch)
    A1 = A[:1]
    C = oracle.emu_gemm("fp16", A1, B, m, n, k)
    Crep = oracle.emu_gemm("fp16", np.repeat(A1, batch, axis=0), B, m, n, k)
    assert np.array_equal(C, Crep)


# ------------------------------------------------------------ f64 / f32 ----
def test_gemm_f64_exact_and_vs_numpy():
    m, n, k = 23, 19, 77
    A, B = _ops(m, n, k, seed=14, dist="int16")
    Ai = np.rint(workloads.math_view(A[0], m)).astype(np.int64)
    Bi = np.rint(workloads.math_view(B[0], k)).astype(np.int64)
    R = workloads.math_view(oracle.gemm_f64(A, B, m, n, k)[0], m)
    assert np.array_equal(R, (Ai @ Bi).astype(np.float64))
    A, B = _ops(m, n, k, seed=15)
    R = workloads.math_view(oracle.gemm_f64(A, B, m, n, k)[0], m)
    ref = workloads.math_view(A[0], m).astype(np.float64) @ workloads.math_view(B[0], k).astype(np.float64)
    assert np.allclose(R, ref, rtol=1e-13, atol=1e-13)


def test_sgemm_f32_exact_and_bound():
    m, n, k = 23, 19, 77
    A, B = _ops(m, n, k, seed=16, dist="int16")
    Ai = np.rint(workloads.math_view(A[0], m)).astype(np.int64)
    Bi = np.rint(workloads.math_view(B[0], k)).astype(np.int64)
    C = workloads.math_view(oracle.sgemm_f32(A, B, m, n, k)[0], m)
    assert np.array_equal(C, (Ai @ Bi).astype(np.float32))
    A, B = _ops(m, n, k, seed=17)
    Am = workloads.math_view(A[0], m).astype(np.float64)
    Bm = workloads.math_view(B[0], k).astype(np.float64)
    exact, _, _ = _exact_product(Am.astype(np.float32)[:4], Bm.astype(np.float32)[:, :4])
    C = workloads.math_view(oracle.sgemm_f32(A, B, m, n, k)[0], m)[:4, :4].astype(np.float64)
    gamma = k * U / (1 - k * U)
    assert np.all(np.abs(C - exact) <= gamma * (np.abs(Am[:4]) @ np.abs(Bm[:, :4])))


def _rn_f32(q):
    """a Fraction rounded to the nearest binary32 (ties to even, subnormals, no
    overflow handling needed here) -- written from the definition"""
    from fractions import Fraction
    if q == 0:
        return 0.0
    neg = q < 0
    a = -q if neg else q
    e = a.numerator.bit_length() - a.denominator.bit_length()
    if Fraction(2) ** e > a:
        e -= 1
    quantum = Fraction(2) ** (max(e, -126) - 23)
    r, rem = divmod(a, quantum)
    if rem > quantum / 2 or (rem == quantum / 2 and r % 2 == 1):
        r += 1
    v = float(r * quantum)
    return -v if neg else v


def test_tf32_ideal_block_sum_is_exact_across_exponents():
    """the ideal model's TF32 block sums (R#9's reference model) are exact sums
    rounded once: with terms 2^120, 2^-70, -2^120 a binary64 running sum would
    lose 2^-70; exponent spreads of 2^+-100 vs Fractions"""
    from fractions import Fraction
    A = np.array([[2.0 ** 60], [1.0], [-(2.0 ** 60)]], dtype=np.float32)        # (k=3, m=1)
    B = np.array([[2.0 ** 60, 2.0 ** -70, 2.0 ** 60]], dtype=np.float32)        # (n=1, k=3)
    assert float(oracle.emu_gemm("tf32", A, B, 1, 1, 3)[0, 0, 0]) == 2.0 ** -70
    rng = np.random.default_rng(77)
    for trial in range(400):
        k = int(rng.integers(1, 17))
        sig = rng.integers(1024, 2048, size=(2, k)).astype(np.float64)
        # wide spreads, and sums in binary32's subnormal range (products 2^-152 .. 2^-120)
        e = rng.integers(-50, 51, size=(2, k)) if trial < 300 else rng.integers(-76, -59, size=(2, k))
        v = (np.ldexp(sig, e - 10) * rng.choice([-1.0, 1.0], size=(2, k))).astype(np.float32)  # TF32-exact
        got = float(oracle.emu_gemm("tf32", v[0].reshape(k, 1), v[1].reshape(1, k), 1, 1, k, kb=64)[0, 0, 0])
        exact = sum((Fraction(float(x)) * Fraction(float(y)) for x, y in zip(v[0], v[1])), Fraction(0))
        assert got == _rn_f32(exact), (trial, got, float(exact))


def test_entry_references_equal_full_references():
    """O4 / O5 at sampled entries (the full-size accuracy gates) are the same
    loops as the full references: equal at every sampled entry, batched, ragged"""
    A, B = workloads.make_operands(3, 37, 29, 53, seed=5)
    g = np.random.default_rng(6)
    b, i, j = g.integers(0, 3, 200), g.integers(0, 37, 200), g.integers(0, 29, 200)
    R = oracle.gemm_f64(A, B, 37, 29, 53)
    S = oracle.sgemm_f32(A, B, 37, 29, 53)
    assert np.array_equal(oracle.gemm_f64_entries(A, B, 37, 29, 53, b, i, j), R[b, j, i])
    assert np.array_equal(oracle.sgemm_f32_entries(A, B, 37, 29, 53, b, i, j), S[b, j, i])
