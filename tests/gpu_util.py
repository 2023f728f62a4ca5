"""GPU-side helpers for the parity tests: run the C ABI on column-major numpy
operands (layout of `workloads`) and compute the element-wise tolerance
 from the oracle's |A||B|."""
import math

import numpy as np

import oracle

U = 2.0 ** -24


def emu_gpu(mode, A, B, m, n, k, alpha=1.0, beta=0.0, C=None, kblock=0, flags=0, range_flag=None,
            ldc=None):
    import torch
    import paper_2308_15152_b200 as emu
    A = np.ascontiguousarray(A, dtype=np.float32)
    B = np.ascontiguousarray(B, dtype=np.float32)
    if A.ndim == 2:
        A = A[None]
    if B.ndim == 2:
        B = B[None]
    batch = max(A.shape[0], B.shape[0])
    lda, ldb = A.shape[2], B.shape[2]
    sA = 0 if (A.shape[0] == 1 and batch > 1) else A.shape[1] * lda
    sB = 0 if (B.shape[0] == 1 and batch > 1) else B.shape[1] * ldb
    ldc = m if ldc is None else ldc
    dA = torch.from_numpy(A).cuda()
    dB = torch.from_numpy(B).cuda()
    if C is None:
        dC = torch.full((batch, n, ldc), float("nan"), device="cuda")
    else:
        dC = torch.from_numpy(np.ascontiguousarray(C, dtype=np.float32).reshape(batch, n, ldc)).cuda()
    emu.emu_sgemm_batched_ex(m, n, k, alpha, dA, lda, sA, dB, ldb, sB, beta, dC, ldc, n * ldc, batch,
                             mode, None, range_flag, kblock, flags)
    torch.cuda.synchronize()
    return dC.cpu().numpy()


def assert_bits_equal(got, want):
    """element-wise equality by value (-0 == +0; NaN == NaN), with a readable
    report of the first mismatches"""
    got = np.asarray(got, dtype=np.float32)
    want = np.asarray(want, dtype=np.float32)
    assert got.shape == want.shape, (got.shape, want.shape)
    bad = ~((got == want) | (np.isnan(got) & np.isnan(want)))
    if np.any(bad):
        idx = np.argwhere(bad)[:5]
        rows = [(tuple(int(v) for v in ix), float(got[tuple(ix)]), float(want[tuple(ix)])) for ix in idx]
        raise AssertionError(f"{int(bad.sum())} of {bad.size} outputs differ from the oracle: {rows}")


def tolerance(mode, A, B, m, n, k, kblock=0):
    """Element-wise bound on |C_gpu - C_oracle|: the tensor
    core's own accumulation of each k-block (at most 2 binary32 ulps per MMA
    instruction of K_inst products plus the block's final alignment), and one
    ulp per cross-block add of the two differently-rounded running sums:
        gamma = 2*(KB/K_inst) + 4 + 2*ceil(k/KB),  tol = gamma * u * (|A||B|)_ij
    """
    kb = kblock or oracle.default_kb(k)
    kinst = 16 if mode in (0, "fp16") else 8
    gamma = 2 * (kb / kinst) + 4 + 2 * math.ceil(max(k, 1) / kb)
    A = np.asarray(A)
    B = np.asarray(B)
    if A.ndim == 2:
        A = A[None]
    if B.ndim == 2:
        B = B[None]
    batch = max(A.shape[0], B.shape[0])
    out = np.empty((batch, n, m))
    for b in range(batch):
        out[b] = oracle.absgemm_f64(A[b if A.shape[0] > 1 else 0], B[b if B.shape[0] > 1 else 0], m, n, k)
    return gamma * U * out


def emu_gpu_range(mode, A, B, m, n, k, alpha=1.0, beta=0.0, C=None, kblock=0, flags=0, range_flag=None):
    """the range-safe entry (R#22) on column-major numpy operands; returns (batch, n, m)"""
    import torch
    import paper_2308_15152_b200 as emu
    A = np.ascontiguousarray(A, dtype=np.float32)
    B = np.ascontiguousarray(B, dtype=np.float32)
    if A.ndim == 2:
        A = A[None]
    if B.ndim == 2:
        B = B[None]
    batch = max(A.shape[0], B.shape[0])
    lda, ldb = A.shape[2], B.shape[2]
    sA = 0 if (A.shape[0] == 1 and batch > 1) else A.shape[1] * lda
    sB = 0 if (B.shape[0] == 1 and batch > 1) else B.shape[1] * ldb
    dA = torch.from_numpy(A).cuda()
    dB = torch.from_numpy(B).cuda()
    if C is None:
        dC = torch.full((batch, n, m), float("nan"), device="cuda")
    else:
        dC = torch.from_numpy(np.ascontiguousarray(C, dtype=np.float32).reshape(batch, n, m)).cuda()
    nbytes = emu.emu_range_workspace_size(m, n, batch)
    ws = torch.empty(max(nbytes // 4, 4), dtype=torch.int32, device="cuda")
    emu.emu_sgemm_batched_range(m, n, k, alpha, dA, lda, sA, dB, ldb, sB, beta, dC, m, n * m, batch,
                                mode, ws, nbytes, None, range_flag, kblock, flags)
    torch.cuda.synchronize()
    return dC.cpu().numpy()
