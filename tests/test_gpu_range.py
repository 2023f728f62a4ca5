"""GPU parity of the range-safe mode (DESIGN R#22):
per-row / per-column power-of-two pre-scaling around the unchanged method,
through emu_sgemm_batched_range, against oracle.emu_gemm_range (pinned in
tests/test_oracle_range.py).  Tolerance: the plain mode's bar of the scaled
problem times 2^(e_i + f_j) (the scaling is exact), plus the final rounding."""
import numpy as np
import pytest

import oracle
import workloads
from gpu_util import assert_bits_equal, emu_gpu, emu_gpu_range, tolerance

pytestmark = pytest.mark.gpu
MODES = ["fp16", "tf32"]


def _cmp(mode, A, B, m, n, k, kblock=0, **kw):
    C = emu_gpu_range(mode, A, B, m, n, k, kblock=kblock, **kw)
    kb = kblock or oracle.default_kb(k)
    ref = oracle.emu_gemm_range(mode, A, B, m, n, k, kb=kb, alpha=kw.get("alpha", 1.0),
                                beta=kw.get("beta", 0.0), C=kw.get("C"), corr=not (kw.get("flags", 0) & 1))
    tol = tolerance(mode, A, B, m, n, k, kb, corr=not (kw.get("flags", 0) & 1), alpha=kw.get("alpha", 1.0),
                    beta=kw.get("beta", 0.0), C=kw.get("C"), range_safe=True)
    d = np.abs(C.astype(np.float64) - ref.astype(np.float64))
    ratio = np.max(d / np.where(tol > 0, tol, 1.0))
    assert np.all(d <= tol), f"max |gpu-oracle|/tol = {ratio:.3g}"
    # bit for bit with the measured tensor-core model (R#9)
    hw = oracle.emu_gemm_range(mode, A, B, m, n, k, kb=kb, alpha=kw.get("alpha", 1.0), beta=kw.get("beta", 0.0),
                               C=kw.get("C"), corr=not (kw.get("flags", 0) & 1), tc="sm100")
    assert_bits_equal(C, hw)
    return C, ref


SHAPES = [
    (1, 256, 256, 1024),     # c4-like magnitudes, square
    (2, 200, 136, 300),      # ragged m, n, k
    (3, 100, 96, 200),       # m <= 128 (the range path always takes the TS kernel)
    (150, 200, 300, 96),     # A-stationary shape
]


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: "x".join(map(str, s)))
def test_range_parity_wide_magnitudes(mode, shape):
    batch, m, n, k = shape
    A, B = workloads.make_operands(batch, m, n, k, seed=500 + m, dist="logu30")
    C, _ = _cmp(mode, A, B, m, n, k)
    assert np.all(np.isfinite(C))


@pytest.mark.parametrize("mode", MODES)
def test_range_policies_and_epilogue(mode):
    batch, m, n, k = 2, 260, 140, 256
    A, B = workloads.make_operands(batch, m, n, k, seed=21, dist="logu30")
    _cmp(mode, A, B, m, n, k, kblock=128)
    _cmp(mode, A, B, m, n, k, flags=1)
    C0 = workloads.uniform((batch, n, m), seed=22)
    _cmp(mode, A, B, m, n, k, alpha=0.75, beta=-1.25, C=C0)   # beta != 0: direct-store epilogue


@pytest.mark.parametrize("mode", MODES)
def test_range_scale_equivariance_bit_exact(mode):
    m, n, k = 256, 128, 512
    A, B = workloads.make_operands(1, m, n, k, seed=23, dist="logu15")
    C = emu_gpu_range(mode, A, B, m, n, k)
    A2 = A.copy()
    A2[0, :, 7] *= np.float32(2.0 ** 9)
    B2 = B.copy()
    B2[0, 5, :] *= np.float32(2.0 ** -11)
    C2 = emu_gpu_range(mode, A2, B2, m, n, k)
    expect = C.copy()
    expect[0, :, 7] *= np.float32(2.0 ** 9)
    expect[0, 5, :] *= np.float32(2.0 ** -11)
    assert np.array_equal(C2, expect)


@pytest.mark.parametrize("mode", MODES)
def test_range_small_integers_exact(mode):
    m, n, k = 300, 260, 1000
    A, B = workloads.make_operands(2, m, n, k, seed=24, dist="int16")
    assert np.array_equal(emu_gpu_range(mode, A, B, m, n, k), oracle.emu_gemm(mode, A, B, m, n, k))


def test_range_equals_plain_when_exponents_zero():
    """rows/columns already peaking in [2^14, 2^15): all exponents 0, the range
    entry and the plain entry run the same kernel on the same values"""
    m, n, k = 256, 256, 320
    A, B = workloads.make_operands(1, m, n, k, seed=25)
    A *= np.float32(2.0 ** 14)
    B *= np.float32(2.0 ** 14)
    for i in range(m):
        A[0, i % k, i] = np.float32(20000.0)
    for j in range(n):
        B[0, j, j % k] = np.float32(-30000.0)
    for mode in MODES:
        assert np.array_equal(emu_gpu_range(mode, A, B, m, n, k), emu_gpu(mode, A, B, m, n, k))


def test_c4_fp16_range_mode():
    """c4 (k = 4096, magnitudes 2^-30..2^30): the plain FP16 mode overflows
    (test_gpu_gemm.test_c4_stress_range); the range-safe FP16 mode passes the
    accuracy gate, stays finite and leaves the range flag clear."""
    import torch
    import paper_2308_15152_b200 as emu
    m = n = 256
    k = 4096
    A, B = workloads.make_operands(1, m, n, k, seed=11, dist="logu30")
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    C = emu_gpu_range("fp16", A, B, m, n, k, range_flag=flag)
    assert emu.emu_last_launch_count() == 2
    assert int(flag.item()) == 0
    assert np.all(np.isfinite(C))
    R = oracle.gemm_f64(A, B, m, n, k)
    e = oracle.rel_frobenius(C, R)
    e_sg = oracle.rel_frobenius(oracle.sgemm_f32(A, B, m, n, k), R)
    assert e <= 2 * e_sg and e <= 1e-5, (e, e_sg)


@pytest.mark.parametrize("mode", MODES)
def test_range_tiny_rows_times_huge_columns(mode):
    """A rows near 2^-100, B columns near 2^120: the result (near 2^20) must be
    finite and accurate -- the unscaling uses the combined exponent, one
    rounding (R#22), never an intermediate (C' * 2^f) that overflows"""
    from test_oracle_range import _tiny_rows_huge_cols
    A, B, m, n, k = _tiny_rows_huge_cols(k=1024, m=200, n=136)
    C, _ = _cmp(mode, A, B, m, n, k)
    assert np.all(np.isfinite(C))
    R = oracle.gemm_f64(A, B, m, n, k)
    assert oracle.rel_frobenius(C, R) <= 2 * oracle.rel_frobenius(oracle.sgemm_f32(A, B, m, n, k), R)
