"""Python binding of the CPU oracle (oracle/oracle.c) -- TEST INFRASTRUCTURE.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this package.  The product package
(paper_2308_15152_b200) never imports it, and it never imports the product.

Arrays follow the column-major storage convention of ``workloads``: an m x k
matrix with leading dimension ld is a float32 array of shape (k, ld);
batched operands are (batch, k, ld).

Functions (each cites the C function that defines it, see oracle.c header):
  split_fp16(x)            -> (hi uint16 bits, lo uint16 bits)    Eqs corr-1..4
  split_tf32(x)            -> (hi float32, lo float32)            reading R#6
  f16_bits_to_f32(bits)    -> float32                             toFP32
  reconstruct(mode, hi, lo)
  emu_gemm(...)            -> C   (emulation model O3)            Eq corr-5
  emu_gemm_entries(...)    -> selected entries of the same model
  gemm_f64(...), absgemm_f64(...), sgemm_f32(...)                 O4 / O5
  rel_frobenius, max_rel_error, componentwise                     metrics O6
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

MODE_FP16 = 0
MODE_TF32 = 1
# "sm100" tensor-core model parameters (R#9): products per aligned
# group, extra alignment bits below the largest term's 24-bit significand
TC_GROUP = 16   # >= K_inst: one fused sum per MMA instruction
TC_EXTRA = 2
TC_JMIN = -158  # lowest bit of the alignment grid (binary32 subnormal quantum 2^-149 / 2^9)
_MODES = {"fp16": MODE_FP16, "tf32": MODE_TF32, MODE_FP16: MODE_FP16, MODE_TF32: MODE_TF32}

BUILD_CMD = ["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math",
             "-fopenmp", "-fPIC", "-shared", "-Wall", "-Wextra", _SRC, "-o", _LIB, "-lm"]


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(BUILD_CMD)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        i64 = ctypes.c_int64
        i32 = ctypes.c_int
        f32 = ctypes.c_float
        f64 = ctypes.c_double
        L.orc_f32_to_f16.argtypes = [f32]; L.orc_f32_to_f16.restype = ctypes.c_uint16
        L.orc_f16_to_f32.argtypes = [ctypes.c_uint16]; L.orc_f16_to_f32.restype = f32
        L.orc_f32_to_tf32.argtypes = [f32]; L.orc_f32_to_tf32.restype = f32
        L.orc_split_fp16.argtypes = [P, i64, P, P]; L.orc_split_fp16.restype = None
        L.orc_split_tf32.argtypes = [P, i64, P, P]; L.orc_split_tf32.restype = None
        L.orc_reconstruct.argtypes = [i32, P, P, i64, P]; L.orc_reconstruct.restype = None
        L.orc_emu_gemm_batched.argtypes = [i32, i32, i32, i32, i32, i32, f32, P, i64, i64,
                                           P, i64, i64, f32, P, i64, i64, i32, i32, i32, i32]
        L.orc_emu_gemm_batched.restype = i32
        L.orc_emu_gemm_entries.argtypes = [i32, i32, i32, i32, i32, i32, f32, P, i64, i64,
                                           P, i64, i64, f32, P, i64, i64, i64, P, P, P, P, i32, i32, i32]
        L.orc_emu_gemm_entries.restype = i32
        L.orc_emu_gemm_range_batched.argtypes = L.orc_emu_gemm_batched.argtypes
        L.orc_emu_gemm_range_batched.restype = i32
        L.orc_emu_gemm_range_entries.argtypes = L.orc_emu_gemm_entries.argtypes
        L.orc_emu_gemm_range_entries.restype = i32
        L.orc_range_exponents.argtypes = [i32, i32, i32, P, i64, P, i64, P, P]
        L.orc_range_exponents.restype = None
        L.orc_gemm_f64_batched.argtypes = [i32, i32, i32, f64, P, i64, i64, P, i64, i64,
                                           f64, P, i64, i64, P, i64, i64, i32]
        L.orc_gemm_f64_batched.restype = None
        L.orc_absgemm_f64.argtypes = [i32, i32, i32, P, i64, P, i64, P, i64]
        L.orc_absgemm_f64.restype = None
        L.orc_sgemm_f32_batched.argtypes = [i32, i32, i32, f32, P, i64, i64, P, i64, i64,
                                            f32, P, i64, i64, i32]
        L.orc_sgemm_f32_batched.restype = None
        L.orc_tc_chain.argtypes = [i32, i32, i32, i32, i32, i32, i32, P, P, P, P]
        L.orc_tc_chain.restype = i32
        L.orc_gemm_f64_entries.argtypes = [i32, P, i64, i64, P, i64, i64, i64, P, P, P, P]
        L.orc_gemm_f64_entries.restype = None
        L.orc_sgemm_f32_entries.argtypes = [i32, P, i64, i64, P, i64, i64, i64, P, P, P, P]
        L.orc_sgemm_f32_entries.restype = None
        L.orc_max_threads.argtypes = []; L.orc_max_threads.restype = i32
        L.orc_set_threads.argtypes = [i32]; L.orc_set_threads.restype = None
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def max_threads() -> int:
    return lib().orc_max_threads()


def set_threads(n: int) -> None:
    lib().orc_set_threads(int(n))


# ---------------------------------------------------------------- split ----
def split_fp16(x):
    x = _f32(x)
    hi = np.empty(x.shape, dtype=np.uint16)
    lo = np.empty(x.shape, dtype=np.uint16)
    lib().orc_split_fp16(_p(x), x.size, _p(hi), _p(lo))
    return hi, lo


def split_tf32(x):
    x = _f32(x)
    hi = np.empty(x.shape, dtype=np.float32)
    lo = np.empty(x.shape, dtype=np.float32)
    lib().orc_split_tf32(_p(x), x.size, _p(hi), _p(lo))
    return hi, lo


def f32_to_f16_bits(x) -> np.ndarray:
    """toFP16 alone (the hi part of the FP16 split)."""
    return split_fp16(x)[0]


def f32_to_tf32(x) -> np.ndarray:
    return split_tf32(x)[0]


def f16_bits_to_f32(bits) -> np.ndarray:
    bits = np.ascontiguousarray(bits, dtype=np.uint16).ravel()
    f = lib().orc_f16_to_f32
    return np.array([f(int(b)) for b in bits], dtype=np.float32)


def split_values(mode, x):
    """split parts as exact float32 values (FP16 parts decoded exactly)."""
    mode = _MODES[mode]
    if mode == MODE_FP16:
        hi, lo = split_fp16(x)
        return _f16_decode(hi), _f16_decode(lo)
    return split_tf32(x)


def _f16_decode(bits):
    # exact decode through the oracle's own toFP32 over the 65536-entry domain
    table = _f16_table()
    return table[np.asarray(bits, dtype=np.uint16)]


_TABLE = None


def _f16_table():
    global _TABLE
    if _TABLE is None:
        _TABLE = f16_bits_to_f32(np.arange(65536, dtype=np.uint32).astype(np.uint16))
    return _TABLE


def reconstruct(mode, hi_val, lo_val):
    mode = _MODES[mode]
    hi_val = _f32(hi_val)
    lo_val = _f32(lo_val)
    out = np.empty(hi_val.shape, dtype=np.float32)
    lib().orc_reconstruct(mode, _p(hi_val), _p(lo_val), hi_val.size, _p(out))
    return out


# ----------------------------------------------------------------- gemm ----
# Tensor-core accumulation models for the block sums of O3 (oracle.c, R#9):
#   "ideal": exact block sum, one RN to binary32;
#   "sm100": per MMA instruction, its products and the accumulator aligned to
#            the largest (un-normalised) exponent with F extra bits (never
#            below 2^J_min), truncated, summed, RZ to binary32 (the paper's RZ,
#            P:495; the parameters fitted by tools/tc_fit.py to the standalone
#            tcgen05 probe's samples, R#9).
#   "simt":  one binary32 FMA per product, k ascending (the device API's
#            CUDA-core policy, R#26).
TC_MODELS = {"ideal": (0, 0, 0), "sm100": (TC_GROUP, TC_EXTRA, TC_JMIN), "simt": (-1, 0, 0)}


def default_kb(k: int) -> int:
    """the library's default combine interval (R#7): 64 for k <= 8192,
    doubled for every further factor 4 of k, at most 4096"""
    kb, lim = 64, 8192
    while k > lim and kb < 4096:
        kb, lim = kb * 2, lim * 4
    return kb


def _check(rc):
    if rc == -2:
        raise ValueError("invalid tensor-core model")
    if rc != 0:
        raise MemoryError("oracle allocation failed")


def tc_chain(mode, A, B, D0=None, tc="sm100"):
    """The tensor-core model at instruction level (oracle.c orc_tc_chain): n
    chained MMA instructions of K_inst = 16 (FP16) / 8 (TF32) exact products.
    A: (n, M, K_inst), B: (n, N, K_inst) exact operand values; D0: (M, N) or
    None.  Returns D (M, N) float32.  `tc` is a TC_MODELS name or a (group,
    extra, jmin) triple (the candidate models of tools/tc_fit.py)."""
    mode = _MODES[mode]
    g, f, jm = TC_MODELS[tc] if isinstance(tc, str) else tc
    A = _f32(A)
    B = _f32(B)
    n, M, K = A.shape
    N = B.shape[1]
    assert K == (16 if mode == MODE_FP16 else 8) and B.shape == (n, N, K)
    D = np.empty((M, N), dtype=np.float32)
    d0 = None if D0 is None else _f32(D0).reshape(M, N)
    _check(lib().orc_tc_chain(mode, g, f, jm, n, M, N, _p(A), _p(B), None if d0 is None else _p(d0), _p(D)))
    return D


def _batched_args(A, B, m, n, k):
    A = _f32(A)
    B = _f32(B)
    if A.ndim == 2:
        A = A[None]
    if B.ndim == 2:
        B = B[None]
    batch = max(A.shape[0], B.shape[0])
    lda = A.shape[2]
    ldb = B.shape[2]
    sA = 0 if A.shape[0] == 1 and batch > 1 else A.shape[1] * A.shape[2]
    sB = 0 if B.shape[0] == 1 and batch > 1 else B.shape[1] * B.shape[2]
    assert A.shape[1] >= k and lda >= m and B.shape[1] >= n and ldb >= k
    return A, B, batch, lda, ldb, sA, sB


def emu_gemm(mode, A, B, m, n, k, alpha=1.0, beta=0.0, C=None, kb=None, corr=True, ldc=None, tc="ideal"):
    """Emulation model O3 over column-major batched operands; returns C as
    (batch, n, ldc) float32.  beta == 0 never reads C."""
    mode = _MODES[mode]
    g, f, jm = TC_MODELS[tc]
    kb = default_kb(k) if not kb else kb
    A, B, batch, lda, ldb, sA, sB = _batched_args(A, B, m, n, k)
    ldc = m if ldc is None else ldc
    if C is None:
        C = np.zeros((batch, n, ldc), dtype=np.float32)
    else:
        C = np.array(C, dtype=np.float32, copy=True).reshape(batch, n, ldc)
    rc = lib().orc_emu_gemm_batched(mode, int(bool(corr)), m, n, k, kb, alpha, _p(A), lda, sA,
                                    _p(B), ldb, sB, beta, _p(C), ldc, n * ldc, batch, g, f, jm)
    _check(rc)
    return C


def emu_gemm_entries(mode, A, B, m, n, k, bidx, ii, jj, alpha=1.0, beta=0.0, C=None,
                     kb=None, corr=True, ldc=None, tc="ideal"):
    mode = _MODES[mode]
    g, f, jm = TC_MODELS[tc]
    kb = default_kb(k) if not kb else kb
    A, B, batch, lda, ldb, sA, sB = _batched_args(A, B, m, n, k)
    ldc = m if ldc is None else ldc
    if C is None:
        C = np.zeros((1, 1, 1), dtype=np.float32)
        sC = 0
    else:
        C = _f32(C)
        sC = n * ldc
    bidx = np.ascontiguousarray(bidx, dtype=np.int64)
    ii = np.ascontiguousarray(ii, dtype=np.int64)
    jj = np.ascontiguousarray(jj, dtype=np.int64)
    out = np.empty(len(ii), dtype=np.float32)
    rc = lib().orc_emu_gemm_entries(mode, int(bool(corr)), m, n, k, kb, alpha, _p(A), lda, sA,
                                    _p(B), ldb, sB, beta, _p(C), ldc, sC, len(ii),
                                    _p(bidx), _p(ii), _p(jj), _p(out), g, f, jm)
    _check(rc)
    return out


def emu_gemm_range(mode, A, B, m, n, k, alpha=1.0, beta=0.0, C=None, kb=None, corr=True, ldc=None, tc="ideal"):
    """Range-safe mode (DESIGN R#22): per-row / per-column
    power-of-two pre-scaling around the unchanged emulation model."""
    mode = _MODES[mode]
    g, f, jm = TC_MODELS[tc]
    kb = default_kb(k) if not kb else kb
    A, B, batch, lda, ldb, sA, sB = _batched_args(A, B, m, n, k)
    ldc = m if ldc is None else ldc
    if C is None:
        C = np.zeros((batch, n, ldc), dtype=np.float32)
    else:
        C = np.array(C, dtype=np.float32, copy=True).reshape(batch, n, ldc)
    rc = lib().orc_emu_gemm_range_batched(mode, int(bool(corr)), m, n, k, kb, alpha, _p(A), lda, sA,
                                          _p(B), ldb, sB, beta, _p(C), ldc, n * ldc, batch, g, f, jm)
    _check(rc)
    return C


def emu_gemm_range_entries(mode, A, B, m, n, k, bidx, ii, jj, alpha=1.0, beta=0.0, C=None,
                           kb=None, corr=True, ldc=None, tc="ideal"):
    mode = _MODES[mode]
    g, f, jm = TC_MODELS[tc]
    kb = default_kb(k) if not kb else kb
    A, B, batch, lda, ldb, sA, sB = _batched_args(A, B, m, n, k)
    ldc = m if ldc is None else ldc
    if C is None:
        C = np.zeros((1, 1, 1), dtype=np.float32)
        sC = 0
    else:
        C = _f32(C)
        sC = n * ldc
    bidx = np.ascontiguousarray(bidx, dtype=np.int64)
    ii = np.ascontiguousarray(ii, dtype=np.int64)
    jj = np.ascontiguousarray(jj, dtype=np.int64)
    out = np.empty(len(ii), dtype=np.float32)
    rc = lib().orc_emu_gemm_range_entries(mode, int(bool(corr)), m, n, k, kb, alpha, _p(A), lda, sA,
                                          _p(B), ldb, sB, beta, _p(C), ldc, sC, len(ii),
                                          _p(bidx), _p(ii), _p(jj), _p(out), g, f, jm)
    _check(rc)
    return out


def range_exponents(A, B, m, n, k):
    """(e_rows[m], f_cols[n]) of one column-major problem (A: (k, lda), B: (n, ldb))."""
    A = _f32(A)
    B = _f32(B)
    e = np.empty(m, dtype=np.int32)
    f = np.empty(n, dtype=np.int32)
    lib().orc_range_exponents(m, n, k, _p(A), A.shape[-1], _p(B), B.shape[-1], _p(e), _p(f))
    return e, f


def gemm_f64(A, B, m, n, k, alpha=1.0, beta=0.0, C=None, ldc=None):
    A, B, batch, lda, ldb, sA, sB = _batched_args(A, B, m, n, k)
    ldc = m if ldc is None else ldc
    R = np.empty((batch, n, m), dtype=np.float64)
    if C is None:
        Cp = np.zeros((1,), dtype=np.float32)
        beta = 0.0
        sC = 0
    else:
        Cp = _f32(C)
        sC = n * ldc
    lib().orc_gemm_f64_batched(m, n, k, alpha, _p(A), lda, sA, _p(B), ldb, sB,
                               beta, _p(Cp), ldc, sC, _p(R), m, n * m, batch)
    return R


def absgemm_f64(A, B, m, n, k):
    """|A||B| in float64 for one (unbatched) product; returns (n, m)."""
    A = _f32(A)
    B = _f32(B)
    R = np.empty((n, m), dtype=np.float64)
    lib().orc_absgemm_f64(m, n, k, _p(A), A.shape[-1], _p(B), B.shape[-1], _p(R), m)
    return R


def sgemm_f32(A, B, m, n, k, alpha=1.0, beta=0.0, C=None, ldc=None):
    A, B, batch, lda, ldb, sA, sB = _batched_args(A, B, m, n, k)
    ldc = m if ldc is None else ldc
    if C is None:
        C = np.zeros((batch, n, ldc), dtype=np.float32)
    else:
        C = np.array(C, dtype=np.float32, copy=True).reshape(batch, n, ldc)
    lib().orc_sgemm_f32_batched(m, n, k, alpha, _p(A), lda, sA, _p(B), ldb, sB,
                                beta, _p(C), ldc, n * ldc, batch)
    return C


def _entries_args(A, B, m, n, k, bidx, ii, jj):
    A, B, batch, lda, ldb, sA, sB = _batched_args(A, B, m, n, k)
    idx = [np.ascontiguousarray(v, dtype=np.int64) for v in (bidx, ii, jj)]
    return A, B, lda, ldb, sA, sB, idx


def gemm_f64_entries(A, B, m, n, k, bidx, ii, jj):
    """O4 (binary64, ascending p) at entries C_{bidx}(ii, jj); alpha = 1, beta = 0"""
    A, B, lda, ldb, sA, sB, idx = _entries_args(A, B, m, n, k, bidx, ii, jj)
    out = np.empty(len(idx[0]), dtype=np.float64)
    lib().orc_gemm_f64_entries(k, _p(A), lda, sA, _p(B), ldb, sB, len(out), *map(_p, idx), _p(out))
    return out


def sgemm_f32_entries(A, B, m, n, k, bidx, ii, jj):
    """O5 (sequential binary32 FMA) at entries C_{bidx}(ii, jj); alpha = 1, beta = 0"""
    A, B, lda, ldb, sA, sB, idx = _entries_args(A, B, m, n, k, bidx, ii, jj)
    out = np.empty(len(idx[0]), dtype=np.float32)
    lib().orc_sgemm_f32_entries(k, _p(A), lda, sA, _p(B), ldb, sB, len(out), *map(_p, idx), _p(out))
    return out


# -------------------------------------------------------------- metrics ----
def rel_frobenius(C, R) -> float:
    """||C - R||_F / ||R||_F (north_star's gate), over finite float64."""
    C = np.asarray(C, dtype=np.float64)
    R = np.asarray(R, dtype=np.float64)
    return float(np.linalg.norm((C - R).ravel()) / np.linalg.norm(R.ravel()))


def max_rel_error(C, R) -> float:
    """max |C - R| / |R| over R != 0 (the paper's metric)."""
    C = np.asarray(C, dtype=np.float64).ravel()
    R = np.asarray(R, dtype=np.float64).ravel()
    nz = R != 0
    return float(np.max(np.abs(C[nz] - R[nz]) / np.abs(R[nz]))) if nz.any() else 0.0


def componentwise(C, R, absAB) -> float:
    """max |C - R| / (u |A||B|), u = 2^-24."""
    C = np.asarray(C, dtype=np.float64)
    R = np.asarray(R, dtype=np.float64)
    d = np.abs(C - R)
    den = np.asarray(absAB, dtype=np.float64) * 2.0 ** -24
    with np.errstate(divide="ignore", invalid="ignore"):
        q = np.where(den > 0, d / den, np.where(d > 0, np.inf, 0.0))
    return float(np.max(q))
