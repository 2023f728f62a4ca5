"""Pins of the oracle's range-safe mode (DESIGN R#22):
per-row (A) / per-column (B) power-of-two pre-scaling around the unchanged
emulation model.  Each pin is fixed by the definition or by the already-pinned
plain model, not by re-typing the oracle's code:

  * exponents: hand-computed values of e = clamp(ilogb(max finite |x|) - 14)
  * operands whose rows/columns already peak in [2^14, 2^15) have all exponents
    0, so the range-safe result equals the plain model bit for bit
  * scaling row i of A (column j of B) by 2^t scales row i (column j) of C by
    exactly 2^t -- catches a missing or sign-flipped un-scaling
  * small integers stay exact (power-of-two scaling loses no bits)
  * the point of the mode: on 2^-30..2^30 operands (c4), where the plain FP16
    split overflows, the accuracy gate (<= 2x FP32 SGEMM, <= 1e-5) holds
"""
import numpy as np
import pytest

import oracle
import workloads


def _col(vals):
    """one column of B (k values) as a (1, k) column-major array, and k"""
    v = np.asarray(vals, dtype=np.float32)
    return v[None, :], len(v)


@pytest.mark.parametrize("vals,expected", [
    ([1.0, -0.5, 0.25], -14),                 # ilogb(1) = 0
    ([65504.0, 1.0], 1),                       # ilogb(65504) = 15
    ([-3.0, 2.0], -13),                        # ilogb(3) = 1
    ([0.0, -0.0, 0.0], 0),                     # no non-zero value
    ([np.inf, 2.0, np.nan], -13),              # non-finite values ignored
    ([np.nan, np.inf], 0),                     # no finite non-zero value
    ([2.0 ** -149], -125),                     # clamp low (ilogb = -149)
    ([2.0 ** 127, 1.0], 113),                  # ilogb = 127
    ([np.float32(2.0 ** 15) - np.float32(2.0 ** 4)], 0),   # 32752 in [2^14, 2^15)
    ([2.0 ** 14], 0),
])
def test_range_exponent_values(vals, expected):
    B, k = _col(vals)
    A = np.zeros((k, 1), dtype=np.float32)
    e, f = oracle.range_exponents(A, B, 1, 1, k)
    assert int(f[0]) == expected
    # the same rule for a row of A
    e2, _ = oracle.range_exponents(np.asarray(vals, dtype=np.float32)[:, None], B, 1, 1, k)
    assert int(e2[0]) == expected


def _peaked(batch, m, n, k, seed):
    """operands whose every row of A and column of B peaks in [2^14, 2^15)"""
    A, B = workloads.make_operands(batch, m, n, k, seed=seed)
    A = A * np.float32(2.0 ** 14)
    B = B * np.float32(2.0 ** 14)
    for b in range(batch):
        for i in range(m):
            A[b, i % k, i] = np.float32(20000.0)
        for j in range(n):
            B[b, j, j % k] = np.float32(-30000.0)
    return A, B


@pytest.mark.parametrize("mode", ["fp16", "tf32"])
def test_range_equals_plain_when_exponents_zero(mode):
    m, n, k = 37, 29, 150
    A, B = _peaked(2, m, n, k, seed=5)
    e, f = oracle.range_exponents(A[0], B[0], m, n, k)
    assert not e.any() and not f.any()
    C0 = workloads.uniform((2, n, m), seed=6)
    for kw in ({}, {"alpha": -1.5, "beta": 0.25, "C": C0}):
        got = oracle.emu_gemm_range(mode, A, B, m, n, k, **kw)
        ref = oracle.emu_gemm(mode, A, B, m, n, k, **kw)
        assert np.array_equal(got, ref)


@pytest.mark.parametrize("mode", ["fp16", "tf32"])
def test_range_scale_equivariance(mode):
    m, n, k = 24, 20, 130
    A, B = workloads.make_operands(1, m, n, k, seed=9, dist="logu15")
    C = oracle.emu_gemm_range(mode, A, B, m, n, k)
    for i, t in ((3, 7), (10, -9), (0, 20)):
        A2 = A.copy()
        A2[0, :, i] *= np.float32(2.0 ** t)
        C2 = oracle.emu_gemm_range(mode, A2, B, m, n, k)
        expect = C.copy()
        expect[0, :, i] *= np.float32(2.0 ** t)
        assert np.array_equal(C2, expect)
    for j, t in ((2, 5), (19, -12)):
        B2 = B.copy()
        B2[0, j, :] *= np.float32(2.0 ** t)
        C2 = oracle.emu_gemm_range(mode, A, B2, m, n, k)
        expect = C.copy()
        expect[0, j, :] *= np.float32(2.0 ** t)
        assert np.array_equal(C2, expect)


@pytest.mark.parametrize("mode", ["fp16", "tf32"])
def test_range_small_integers_exact(mode):
    m, n, k = 33, 17, 300
    A, B = workloads.make_operands(2, m, n, k, seed=8, dist="int16")
    exact = np.einsum("bkm,bnk->bnm", A.astype(np.float64), B.astype(np.float64))
    assert np.array_equal(oracle.emu_gemm_range(mode, A, B, m, n, k).astype(np.float64), exact)


@pytest.mark.parametrize("mode", ["fp16", "tf32"])
def test_range_accuracy_gate_wide_magnitudes(mode):
    """c4-style operands (|x| in 2^-30..2^30): the plain FP16 split overflows
    (R#4); the range-safe mode meets north_star's gate."""
    m = n = 48
    k = 1024
    A, B = workloads.make_operands(1, m, n, k, seed=11, dist="logu30")
    R = oracle.gemm_f64(A, B, m, n, k)
    e_sg = oracle.rel_frobenius(oracle.sgemm_f32(A, B, m, n, k), R)
    C = oracle.emu_gemm_range(mode, A, B, m, n, k)
    assert np.all(np.isfinite(C))
    e = oracle.rel_frobenius(C, R)
    assert e <= 2 * e_sg and e <= 1e-5, (e, e_sg)
    if mode == "fp16":
        assert not np.all(np.isfinite(oracle.emu_gemm("fp16", A, B, m, n, k)))


def test_range_entries_match_full():
    m, n, k = 40, 36, 200
    A, B = workloads.make_operands(3, m, n, k, seed=13, dist="logu30")
    C0 = workloads.uniform((3, n, m), seed=14)
    full = oracle.emu_gemm_range("fp16", A, B, m, n, k, alpha=0.5, beta=2.0, C=C0)
    g = workloads.rng(15)
    b, i, j = g.integers(0, 3, 64), g.integers(0, m, 64), g.integers(0, n, 64)
    got = oracle.emu_gemm_range_entries("fp16", A, B, m, n, k, b, i, j, alpha=0.5, beta=2.0, C=C0)
    assert np.array_equal(got, full[b, j, i])


def _tiny_rows_huge_cols(k=1024, m=24, n=20, seed=77):
    """rows of A near 2^-100 and columns of B near 2^120 (some rows / columns
    at ordinary magnitudes): the entries of A B lie near 2^20, well inside
    binary32, but (C' * 2^f) alone would overflow -- the case the combined
    exponent of R#22 exists for (round-2 advisor finding)"""
    g = workloads.rng(seed)
    A = g.uniform(-1, 1, size=(1, k, m)).astype(np.float32)
    B = g.uniform(-1, 1, size=(1, n, k)).astype(np.float32)
    A[:, :, : m - 4] *= np.float32(2.0 ** -100)
    B[:, : n - 3, :] *= np.float32(2.0 ** 120)
    return A, B, m, n, k


@pytest.mark.parametrize("mode", ["fp16", "tf32"])
def test_range_tiny_rows_times_huge_columns(mode):
    A, B, m, n, k = _tiny_rows_huge_cols()
    e, f = oracle.range_exponents(A[0], B[0], m, n, k)
    assert e.min() <= -113 and f.max() >= 105           # the scaling really is extreme
    C = oracle.emu_gemm_range(mode, A, B, m, n, k)
    assert np.all(np.isfinite(C))
    R = oracle.gemm_f64(A, B, m, n, k)
    assert oracle.rel_frobenius(C, R) <= 2 * oracle.rel_frobenius(oracle.sgemm_f32(A, B, m, n, k), R)
