"""Structured operands of the paper's primitive-function benchmarks, written
out as explicit FP32 matrices -- TEST INFRASTRUCTURE (same import rule as the
rest of ``oracle``: only tests/, smoke() and bench.py's CPU legs use it).

The device API generates these operands inside the kernel (foreach_ij / map
analogs, include/emu_tcec.cuh); here they are built plainly, element by
element as the paper's code fragments state, and then multiplied with the
oracle's emulation model ``oracle.emu_gemm`` (O3).  Matrices are returned as
the m x m MATH view (float32, row index = i); ``workloads.colmajor`` turns
them into the column-major storage the GEMM oracle takes.

  householder_matrix(v)   H = I - 2 v v^T, H(i,p) = RN(RN(RN(v_i v_p) * -2) + [i == p])
                          Eq. householder with Code 4's element rule
                          (elm = v[i]*v[j]*(-2); if (i==j) elm += 1);
                          DESIGN R#23 (the paper prints v^T v; v v^T is meant)
  givens_matrix(m,i,j,c,s) G(i, j, theta) of P:416-437 (DESIGN R#24)
  scan_matrix(n)          L = U^T, L(i, p) = [p <= i]: Eqs. scan-mat / u-rule
                           for column arrays (DESIGN R#25)
"""
from __future__ import annotations

import numpy as np

__all__ = ["householder_matrix", "givens_matrix", "scan_matrix"]


def householder_matrix(v) -> np.ndarray:
    """Code 4's element rule in binary32: each product v_i*v_p rounded once
    (numpy float32 multiply), the *(-2) exact, then +1 on the diagonal
    rounded once.  Returns (m, m) float32."""
    v = np.asarray(v, dtype=np.float32)
    m = v.shape[0]
    H = np.empty((m, m), dtype=np.float32)
    for i in range(m):
        row = v[i] * v                         # float32 * float32 -> float32, RN
        row = row * np.float32(-2.0)           # exact
        row[i] = row[i] + np.float32(1.0)      # RN
        H[i] = row
    return H


def givens_matrix(m: int, i: int, j: int, c: float, s: float) -> np.ndarray:
    """G(i, j, theta): identity except G(i,i) = G(j,j) = c, G(i,j) = -s,
    G(j,i) = s (the matrix printed at P:422-434; rows/columns i and j)."""
    assert 0 <= i < m and 0 <= j < m and i != j
    G = np.eye(m, dtype=np.float32)
    G[i, i] = np.float32(c)
    G[j, j] = np.float32(c)
    G[i, j] = -np.float32(s)
    G[j, i] = np.float32(s)
    return G


def scan_matrix(n: int) -> np.ndarray:
    """L(i, p) = 1 if p <= i else 0, so (L x)_i = sum_{p <= i} x_p -- the
    transpose of the paper's U (u_{i,j} = 1 for i <= j, Eq. u-rule), applied
    to column arrays instead of row vectors (a^T U = (L a)^T)."""
    L = np.zeros((n, n), dtype=np.float32)
    for i in range(n):
        L[i, : i + 1] = 1.0
    return L
