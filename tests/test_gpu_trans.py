"""GPU parity of op(A) / op(B) transposes (emu_sgemm_batched_t, SURVEY §8(f)
NEXT 2).  The transposed operand is only read differently (TMA box and the
splitters' shared-memory reads); the split values, MMAs and combine are the
same, so a transposed call is bit-identical to the plain call on the explicitly
transposed copy, and both match the oracle on that copy."""
import numpy as np
import pytest

import oracle
import workloads
from gpu_util import emu_gpu, tolerance

pytestmark = pytest.mark.gpu
MODES = ["fp16", "tf32"]


def _stored_t(X):
    """column-major (batch, c, ld) of an r x c matrix -> storage of its transpose
    (c x r column-major: (batch, r, ld') with ld' the next multiple of 4 above c),
    padding filled with NaN (never read)"""
    b, c, ld = X.shape
    r = ld
    out = np.full((b, r, c + 4 - c % 4), np.nan, dtype=np.float32)
    out[:, :, :c] = np.transpose(X, (0, 2, 1))
    return out


def _gpu_t(mode, ta, tb, As, Bs, m, n, k, **kw):
    import torch
    import paper_2308_15152_b200 as emu
    batch = max(As.shape[0], Bs.shape[0])
    lda, ldb = As.shape[2], Bs.shape[2]
    dA = torch.from_numpy(np.ascontiguousarray(As)).cuda()
    dB = torch.from_numpy(np.ascontiguousarray(Bs)).cuda()
    C0 = kw.get("C")
    dC = (torch.full((batch, n, m), float("nan"), device="cuda") if C0 is None
          else torch.from_numpy(np.ascontiguousarray(C0, dtype=np.float32)).cuda())
    emu.emu_sgemm_batched_t(ta, tb, m, n, k, kw.get("alpha", 1.0), dA, lda, As.shape[1] * lda, dB, ldb,
                            Bs.shape[1] * ldb, kw.get("beta", 0.0), dC, m, n * m, batch, mode,
                            kblock=kw.get("kblock", 0))
    torch.cuda.synchronize()
    return dC.cpu().numpy()


SHAPES = [
    (2, 200, 136, 300),      # ragged m, n, k
    (3, 256, 256, 256),      # c2 item shape
    (150, 200, 300, 96),     # A-stationary
    (4, 100, 60, 70),        # m <= 128 (transposes always take the TS kernel)
]


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("trans", ["TN", "NT", "TT"])
@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: "x".join(map(str, s)))
def test_transposed_parity(mode, trans, shape):
    batch, m, n, k = shape
    # op(A): (batch, k, lda), op(B): (batch, n, ldb); leading dimensions in the TMA domain
    A, B = workloads.make_operands(batch, m, n, k, seed=700 + m + n, lda=-(-m // 4) * 4, ldb=-(-k // 4) * 4)
    As = _stored_t(A) if trans[0] == "T" else A
    Bs = _stored_t(B) if trans[1] == "T" else B
    C = _gpu_t(mode, trans[0], trans[1], As, Bs, m, n, k)
    ref = oracle.emu_gemm(mode, A, B, m, n, k)
    tol = tolerance(mode, A, B, m, n, k)
    assert np.all(np.abs(C.astype(np.float64) - ref) <= tol)
    if m > 128:   # the plain call takes the same TS kernel: identical bits
        assert np.array_equal(C, emu_gpu(mode, A, B, m, n, k))


@pytest.mark.parametrize("mode", MODES)
def test_transposed_exact_and_epilogue(mode):
    m, n, k, batch = 300, 260, 1000, 2
    A, B = workloads.make_operands(batch, m, n, k, seed=8, dist="int16")
    C0 = workloads.small_int((batch, n, m), seed=9)
    exact = oracle.emu_gemm(mode, A, B, m, n, k, beta=1.0, C=C0)
    got = _gpu_t(mode, "T", "T", _stored_t(A), _stored_t(B), m, n, k, beta=1.0, C=C0)
    assert np.array_equal(got, exact)
    A, B = workloads.make_operands(1, m, n, k, seed=10)
    got = _gpu_t(mode, "T", "N", _stored_t(A), B, m, n, k, kblock=128)
    assert np.array_equal(got, emu_gpu(mode, A, B, m, n, k, kblock=128))
