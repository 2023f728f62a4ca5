"""Pins of the oracle's "sm100" tensor-core accumulation model (oracle.c
tc_instr, R#9) against what the paper and the mathematics fix:

* P:495 / S:213: the Tensor Core's own accumulation rounds toward zero --
  1 + 3*2^-24 (one instruction) gives 1 + 2^-23 (RZ), where the "ideal" model
  (one RN of the exact block sum) gives 1 + 2^-22;
* exactness: identity / permutation operands and small integers reach the
  exact result (every term lies on the alignment grid);
* truncation only: with all terms positive, the model never exceeds the exact
  sum and stays within the derived alignment + RZ bound below it; with signs,
  |model - exact| stays within the same bound;
* odd symmetry: negating A negates C bit for bit (RZ is symmetric).
Exact sums are Python Fractions (independent of oracle.c)."""
import math
from fractions import Fraction

import numpy as np
import pytest

import oracle


def _dot_model(mode, a, b, kb=64):
    k = len(a)
    A = np.asarray(a, dtype=np.float32).reshape(k, 1)
    B = np.asarray(b, dtype=np.float32).reshape(1, k)
    return float(oracle.emu_gemm(mode, A, B, 1, 1, k, kb=kb, tc="sm100")[0, 0, 0])


@pytest.mark.parametrize("mode", ["fp16", "tf32"])
def test_paper_rz_vector(mode):
    K = 16 if mode == "fp16" else 8
    a = [1.0, 3 * 2.0 ** -12] + [0.0] * (K - 2)
    b = [1.0, 2.0 ** -12] + [0.0] * (K - 2)
    assert _dot_model(mode, a, b) == 1 + 2.0 ** -23          # RZ
    assert _dot_model(mode, [-x for x in a], b) == -(1 + 2.0 ** -23)
    A = np.asarray(a, dtype=np.float32).reshape(K, 1)
    B = np.asarray(b, dtype=np.float32).reshape(1, K)
    assert float(oracle.emu_gemm(mode, A, B, 1, 1, K, tc="ideal")[0, 0, 0]) == 1 + 2.0 ** -22   # RN


@pytest.mark.parametrize("mode", ["fp16", "tf32"])
def test_identity_and_permutation_exact(mode):
    rng = np.random.default_rng(5)
    m = 48
    B = rng.uniform(-1, 1, size=(m, m)).astype(np.float32)   # (n, k) column-major k x n
    P = np.eye(m, dtype=np.float32)[rng.permutation(m)]
    hi, lo = oracle.split_values(mode, B)
    want = oracle.reconstruct(mode, hi, lo)
    for A in (np.eye(m, dtype=np.float32), P):
        C = oracle.emu_gemm(mode, A, B, m, m, m, tc="sm100")[0]
        # C(i, j) = sum_p A(i, p) B(p, j) = B(p_i, j); A stored (k, m): A[p, i] = A(i, p)
        idx = np.argmax(A, axis=0)     # for each i, the p with A(i, p) = 1
        np.testing.assert_array_equal(C, want[:, idx])


@pytest.mark.parametrize("mode", ["fp16", "tf32"])
@pytest.mark.parametrize("k", [7, 64, 300])
def test_small_integers_exact(mode, k):
    rng = np.random.default_rng(k)
    m, n = 9, 11
    A = rng.integers(-16, 17, size=(k, m)).astype(np.float32)
    B = rng.integers(-16, 17, size=(n, k)).astype(np.float32)
    C = oracle.emu_gemm(mode, A, B, m, n, k, tc="sm100")[0]
    exact = (B.astype(np.int64) @ A.astype(np.int64))       # (n, m): sum_p B(p, j) A(i, p)
    np.testing.assert_array_equal(C, exact.astype(np.float32))


@pytest.mark.parametrize("mode", ["fp16", "tf32"])
def test_truncation_only_positive_terms(mode):
    """All terms positive and exactly representable (lo = 0): the model is
    below the exact sum (only truncations), and within the bound: per group
    of G products, each of the G + 1 truncated terms loses < 2^(e_max-23-F)
    <= 2^(-23-F) * S (S = the running sum, which bounds e_max) and the RZ
    loses < 2^-23 * S, so exact - model <= n_groups * ((G+1) 2^-F + 1) 2^-23 S."""
    rng = np.random.default_rng(11)
    K = 16 if mode == "fp16" else 8
    G, F, _ = oracle.TC_MODELS["sm100"]
    for trial in range(200):
        k = int(rng.integers(1, 65))
        sig = rng.integers(1024, 2048, size=(2, k)).astype(np.float64)
        e = rng.integers(-6, 7, size=(2, k))
        v = np.ldexp(sig, e - 10).astype(np.float32)
        got = Fraction(_dot_model(mode, v[0], v[1]))
        exact = sum((Fraction(float(x)) * Fraction(float(y)) for x, y in zip(v[0], v[1])), Fraction(0))
        groups = sum(math.ceil(min(K, k - s) / G) for s in range(0, k, K))
        bound = groups * ((G + 1) * Fraction(1, 2 ** F) + 1) * Fraction(1, 2 ** 23) * exact
        assert got <= exact, (trial, float(got), float(exact))
        assert exact - got <= bound, (trial, float(exact - got), float(bound))


@pytest.mark.parametrize("mode", ["fp16", "tf32"])
def test_signed_terms_bound_and_odd_symmetry(mode):
    """Mixed signs (cancellation): per group the error is < (G+1) 2^(e_max-23-F)
    + 2^-23 |result| with 2^e_max <= the largest term magnitude <= the sum of
    |terms| (running |sum| included), so |model - exact| <= n_groups ((G+1) 2^-F
    + 1) 2^-23 * (sum |products| + |partial sums|) <= 2 n_groups (...) sum|p|."""
    rng = np.random.default_rng(12)
    K = 16 if mode == "fp16" else 8
    G, F, _ = oracle.TC_MODELS["sm100"]
    for trial in range(200):
        k = int(rng.integers(1, 65))
        sig = rng.integers(1024, 2048, size=(2, k)).astype(np.float64)
        e = rng.integers(-6, 7, size=(2, k))
        s = rng.choice([-1.0, 1.0], size=(2, k))
        v = (np.ldexp(sig, e - 10) * s).astype(np.float32)
        got = _dot_model(mode, v[0], v[1])
        assert _dot_model(mode, -v[0], v[1]) == -got
        exact = sum((Fraction(float(x)) * Fraction(float(y)) for x, y in zip(v[0], v[1])), Fraction(0))
        absum = sum((abs(Fraction(float(x)) * Fraction(float(y))) for x, y in zip(v[0], v[1])), Fraction(0))
        groups = sum(math.ceil(min(K, k - s0) / G) for s0 in range(0, k, K))
        bound = 2 * groups * ((G + 1) * Fraction(1, 2 ** F) + 1) * Fraction(1, 2 ** 23) * absum
        assert abs(Fraction(got) - exact) <= bound, (trial, got, float(exact))


@pytest.mark.parametrize("mode", ["fp16", "tf32"])
@pytest.mark.parametrize("k", [200, 4096, 16384])
def test_general_inputs_within_gpu_tolerance(mode, k):
    """The sm100 model stays within the element-wise bar the GPU parity tests
    use against the ideal model (tests/gpu_util.py entry_bound),
    and the bar discriminates: dropping the correction products, or doubling
    their 2^-11 scale (C_on + (C_on - C_off)), exceeds it at every k."""
    from gpu_util import tolerance_entries
    rng = np.random.default_rng(13)
    m = n = 24
    A = rng.uniform(-1, 1, size=(1, k, m)).astype(np.float32)
    B = rng.uniform(-1, 1, size=(1, n, k)).astype(np.float32)
    b = np.zeros(32, dtype=np.int64)
    i, j = rng.integers(0, m, 32), rng.integers(0, n, 32)
    ideal = oracle.emu_gemm_entries(mode, A, B, m, n, k, b, i, j, tc="ideal").astype(np.float64)
    hw = oracle.emu_gemm_entries(mode, A, B, m, n, k, b, i, j, tc="sm100").astype(np.float64)
    off = oracle.emu_gemm_entries(mode, A, B, m, n, k, b, i, j, tc="sm100", corr=False).astype(np.float64)
    tol = tolerance_entries(mode, A, B, k, b, i, j)
    assert np.all(np.abs(hw - ideal) <= tol)
    assert np.any(hw != ideal)          # the two models really differ on general inputs
    assert np.mean(np.abs(off - ideal) > tol) > 0.5
    assert np.mean(np.abs(2 * hw - off - ideal) > tol) > 0.5


@pytest.mark.parametrize("mode", ["fp16", "tf32"])
def test_simt_model_is_sequential_fma_sgemm(mode):
    """the "simt" model (R#26) on operands exactly representable in the split
    format (lo = 0) and k <= KB is the textbook sequential-FMA SGEMM (O5)"""
    rng = np.random.default_rng(14)
    m, n, k = 10, 9, 64
    sig = rng.integers(1024, 2048, size=(2, k * max(m, n))).astype(np.float64)
    e = rng.integers(-5, 6, size=sig.shape)
    v = (np.ldexp(sig, e - 10) * rng.choice([-1.0, 1.0], size=sig.shape)).astype(np.float32)
    A = v[0, :k * m].reshape(k, m)
    B = v[1, :k * n].reshape(n, k)
    got = oracle.emu_gemm(mode, A, B, m, n, k, tc="simt")
    np.testing.assert_array_equal(got, oracle.sgemm_f32(A, B, m, n, k))


def test_default_kb_table():
    """R#7's default combine interval, as documented in include/emu_sgemm.h"""
    table = {1: 64, 4096: 64, 8192: 64, 8193: 128, 16384: 128, 32768: 128, 32769: 256,
             131072: 256, 131073: 512}
    for k, kb in table.items():
        assert oracle.default_kb(k) == kb, k
