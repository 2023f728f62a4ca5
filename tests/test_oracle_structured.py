"""Pins for oracle/structured.py (the explicit Householder, Givens and scan
operands of P:311-470) against things other than itself: an exact-rational
evaluation of Code 4's element rule, orthogonality and the
reflection / rotation identities of the exact matrices, and exact prefix sums.
"""
import fractions
import math

import numpy as np
import pytest

import oracle
import workloads
from oracle import structured

U = 2.0 ** -24
F = fractions.Fraction


def rn32(q: F) -> float:
    """round-to-nearest-even of a rational to binary32 (subnormals included)."""
    if q == 0:
        return 0.0
    s = -1 if q < 0 else 1
    a = abs(q)
    e = a.numerator.bit_length() - a.denominator.bit_length()
    if F(2) ** e > a:
        e -= 1
    ulp = F(2) ** (max(e, -126) - 23)
    return s * float(round(a / ulp) * ulp)   # round(Fraction) is half-to-even


def test_householder_rule_exact():
    """H(i,p) == RN(RN(v_i v_p) * -2 + [i == p]) evaluated in exact rationals."""
    v = workloads.unit_vectors(1, 11, seed=3)[0]
    H = structured.householder_matrix(v)
    for i in range(11):
        for p in range(11):
            e = F(rn32(F(float(v[i])) * F(float(v[p])))) * -2
            expect = rn32(e + (1 if i == p else 0))
            assert float(H[i, p]) == expect, (i, p)


def test_householder_reflection_identities():
    """H = I - 2vv^T with ||v|| = 1: H H^T = I, H v = -v, H w = w for w _|_ v
    (up to the rounding of v and of each element: a few u)."""
    m = 40
    v = workloads.unit_vectors(1, m, seed=8)[0]
    H = structured.householder_matrix(v).astype(np.float64)
    v64 = v.astype(np.float64)
    assert np.max(np.abs(H @ H.T - np.eye(m))) <= 8 * m * U
    assert np.max(np.abs(H @ v64 + v64)) <= 8 * m * U
    w = workloads.uniform(m, seed=9).astype(np.float64)
    w -= v64 * (v64 @ w) / (v64 @ v64)
    assert np.max(np.abs(H @ w - w)) <= 8 * m * U * np.max(np.abs(w))
    assert np.allclose(H, H.T, rtol=0, atol=0)     # the rule is symmetric in (i, p)


def test_givens_rotation_identities():
    m, i, j = 20, 3, 17
    c, s = workloads.rotations(1, seed=4)[0]
    G = structured.givens_matrix(m, i, j, c, s)
    G64 = G.astype(np.float64)
    assert np.max(np.abs(G64 @ G64.T - np.eye(m))) <= 4 * U
    e = np.zeros(m)
    e[i] = 1.0
    y = G64 @ e                      # column i: c at row i, s at row j
    assert y[i] == c and y[j] == s and np.count_nonzero(y) == 2
    assert np.array_equal(structured.givens_matrix(m, i, j, 1.0, 0.0), np.eye(m, dtype=np.float32))


def test_scan_matrix_prefix_sums():
    n = 37
    x = workloads.small_int(n, seed=2).astype(np.float64)
    L = structured.scan_matrix(n).astype(np.float64)
    assert np.array_equal(L @ x, np.cumsum(x))
    assert np.array_equal(L, np.tril(np.ones((n, n))))


@pytest.mark.parametrize("mode", ["fp16", "tf32"])
def test_householder_through_emulation_accuracy(mode):
    """the emulation model applied to the explicit H reaches FP32-SGEMM accuracy
    against the exact reflection in float64 (P:557 claim, structured operand)."""
    m, n = 96, 24
    v = workloads.unit_vectors(1, m, seed=12)[0]
    H = structured.householder_matrix(v)
    _, X = workloads.make_operands(1, n, n, m, seed=13)      # X: (1, n, m) = m x n column-major
    Hc = workloads.colmajor(H)[None]
    C = oracle.emu_gemm(mode, Hc, X, m, n, m)
    R = oracle.gemm_f64(Hc, X, m, n, m)
    e_emu = oracle.rel_frobenius(C, R)
    e_sg = oracle.rel_frobenius(oracle.sgemm_f32(Hc, X, m, n, m), R)
    assert e_emu <= 2 * e_sg + 1e-8 and e_emu <= 1e-5
    assert math.isfinite(e_emu)
