"""Python binding of libemusgemm.so -- the B200 emulated-SGEMM C ABI
(include/emu_sgemm.h).  Argument marshalling only: every step of the method
runs in the library's sm_100a kernels.  There is no fallback: if the library
is missing this import fails.

Functions keep the C names and argument order; pointer arguments accept a
torch tensor (its data_ptr()), an int address or None.  `stream` defaults to
torch's current CUDA stream.  A non-SUCCESS status raises EmuError.
"""
from __future__ import annotations

import ctypes
import os

__all__ = [
    "EMU_SPLIT_FP16", "EMU_SPLIT_TF32", "EMU_FLAG_NO_CORRECTION", "EmuError", "lib", "LIB_PATH",
    "emu_sgemm", "emu_sgemm_batched", "emu_sgemm_batched_ex", "emu_sgemm_batched_host",
    "emu_split", "emu_status_string", "emu_version", "emu_last_launch_count", "emu_last_kernel_name", "mode_of",
    "EMU_FLAG_SIMT", "EMU_FLAG_PIPELINED", "emu_tcec_gemm_batched", "emu_tcec_householder_batched", "emu_tcec_givens_batched",
    "emu_tcec_scan", "emu_sgemm_multicast", "EMU_COL_MAJOR", "EMU_ROW_MAJOR", "emu_sgemm_batched_layout",
    "matmul",
]

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libemusgemm.so")

EMU_SPLIT_FP16 = 0
EMU_SPLIT_TF32 = 1
EMU_FLAG_NO_CORRECTION = 1
EMU_FLAG_SIMT = 2
EMU_FLAG_PIPELINED = 4
EMU_COL_MAJOR = 0
EMU_ROW_MAJOR = 1
STATUS = {0: "SUCCESS", 1: "INVALID_VALUE", 2: "NOT_SUPPORTED", 3: "ARCH_MISMATCH",
          4: "LAUNCH_FAILED", 5: "CUDA_ERROR"}


class EmuError(RuntimeError):
    def __init__(self, status: int, where: str):
        super().__init__(f"{where}: EMU_STATUS_{STATUS.get(status, status)}")
        self.status = status


if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is not built; run `python -m paper_2308_15152_b200.build` "
                      "(or __graft_entry__.build()). There is no CPU fallback.")

lib = ctypes.CDLL(LIB_PATH)
_i = ctypes.c_int
_ll = ctypes.c_longlong
_f = ctypes.c_float
_p = ctypes.c_void_p
_u = ctypes.c_uint

_GEMM_ARGS = [_i, _i, _i, _f, _p, _i, _ll, _p, _i, _ll, _f, _p, _i, _ll, _i, _i, _p]
lib.emu_sgemm_batched.argtypes = _GEMM_ARGS
lib.emu_sgemm_batched.restype = _i
lib.emu_sgemm_batched_ex.argtypes = _GEMM_ARGS + [_p, _i, _u]
lib.emu_sgemm_batched_ex.restype = _i
lib.emu_sgemm_batched_t.argtypes = [ctypes.c_char, ctypes.c_char] + _GEMM_ARGS + [_p, _i, _u]
lib.emu_sgemm_batched_t.restype = _i
lib.emu_sgemm_batched_range.argtypes = _GEMM_ARGS + [_p, ctypes.c_size_t, _p, _i, _u]
lib.emu_sgemm_batched_range.restype = _i
lib.emu_range_workspace_size.argtypes = [_i, _i, _i]
lib.emu_range_workspace_size.restype = ctypes.c_size_t
lib.emu_sgemm_batched_host.argtypes = _GEMM_ARGS
lib.emu_sgemm_batched_host.restype = _i
lib.emu_sgemm.argtypes = [_i, _i, _i, _f, _p, _i, _p, _i, _f, _p, _i, _i, _p]
lib.emu_sgemm.restype = _i
lib.emu_split.argtypes = [_p, _ll, _i, _p, _p, _p]
lib.emu_split.restype = _i
lib.emu_tcec_gemm_batched.argtypes = _GEMM_ARGS + [_i, _u]
lib.emu_tcec_gemm_batched.restype = _i
lib.emu_tcec_householder_batched.argtypes = [_i, _i, _p, _ll, _p, _i, _ll, _p, _i, _ll, _i, _i, _p, _u]
lib.emu_tcec_householder_batched.restype = _i
lib.emu_tcec_givens_batched.argtypes = [_i, _i, _i, _i, _p, _p, _i, _ll, _p, _i, _ll, _i, _i, _p, _u]
lib.emu_tcec_givens_batched.restype = _i
lib.emu_tcec_scan.argtypes = [_i, _i, _p, _i, _p, _i, _i, _p, _u]
lib.emu_tcec_scan.restype = _i
lib.emu_sgemm_batched_layout.argtypes = [_i, ctypes.c_char, ctypes.c_char] + _GEMM_ARGS + [_p, _i, _u]
lib.emu_sgemm_batched_layout.restype = _i
lib.emu_sgemm_multicast.argtypes = [_i, _i, _i, _f, _p, _i, _p, _i, ctypes.POINTER(_p), _i, _i, _i, _p, _i, _u]
lib.emu_sgemm_multicast.restype = _i
lib.emu_status_string.argtypes = [_i]
lib.emu_status_string.restype = ctypes.c_char_p
lib.emu_version.argtypes = []
lib.emu_version.restype = _i
lib.emu_last_launch_count.argtypes = []
lib.emu_last_launch_count.restype = _i
lib.emu_last_kernel_name.argtypes = []
lib.emu_last_kernel_name.restype = ctypes.c_char_p


def mode_of(mode) -> int:
    if mode in (EMU_SPLIT_FP16, "fp16"):
        return EMU_SPLIT_FP16
    if mode in (EMU_SPLIT_TF32, "tf32"):
        return EMU_SPLIT_TF32
    return int(mode)  # let the library reject it


def _ptr(x):
    if x is None:
        return None
    if isinstance(x, int):
        return x
    if hasattr(x, "data_ptr"):
        return x.data_ptr()
    if hasattr(x, "ctypes"):          # numpy array (host entry)
        return x.ctypes.data
    raise TypeError(type(x))


def _stream(s):
    if s is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    if isinstance(s, int):
        return s
    return s.cuda_stream


def _check(st: int, where: str):
    if st != 0:
        raise EmuError(st, where)


def emu_sgemm_batched(m, n, k, alpha, A, lda, strideA, B, ldb, strideB, beta, C, ldc, strideC,
                      batch, mode, stream=None):
    _check(lib.emu_sgemm_batched(m, n, k, alpha, _ptr(A), lda, strideA, _ptr(B), ldb, strideB,
                                 beta, _ptr(C), ldc, strideC, batch, mode_of(mode), _stream(stream)),
           "emu_sgemm_batched")


def emu_sgemm_batched_ex(m, n, k, alpha, A, lda, strideA, B, ldb, strideB, beta, C, ldc, strideC,
                         batch, mode, stream=None, range_flag=None, kblock=0, flags=0):
    _check(lib.emu_sgemm_batched_ex(m, n, k, alpha, _ptr(A), lda, strideA, _ptr(B), ldb, strideB,
                                    beta, _ptr(C), ldc, strideC, batch, mode_of(mode), _stream(stream),
                                    _ptr(range_flag), kblock, flags),
           "emu_sgemm_batched_ex")


def emu_sgemm_batched_t(transa, transb, m, n, k, alpha, A, lda, strideA, B, ldb, strideB, beta, C, ldc,
                        strideC, batch, mode, stream=None, range_flag=None, kblock=0, flags=0):
    _check(lib.emu_sgemm_batched_t(transa.encode() if isinstance(transa, str) else transa,
                                   transb.encode() if isinstance(transb, str) else transb,
                                   m, n, k, alpha, _ptr(A), lda, strideA, _ptr(B), ldb, strideB,
                                   beta, _ptr(C), ldc, strideC, batch, mode_of(mode), _stream(stream),
                                   _ptr(range_flag), kblock, flags),
           "emu_sgemm_batched_t")


def emu_range_workspace_size(m, n, batch) -> int:
    return int(lib.emu_range_workspace_size(m, n, batch))


def emu_sgemm_batched_range(m, n, k, alpha, A, lda, strideA, B, ldb, strideB, beta, C, ldc, strideC,
                            batch, mode, workspace, workspace_bytes, stream=None, range_flag=None, kblock=0,
                            flags=0):
    _check(lib.emu_sgemm_batched_range(m, n, k, alpha, _ptr(A), lda, strideA, _ptr(B), ldb, strideB,
                                       beta, _ptr(C), ldc, strideC, batch, mode_of(mode), _stream(stream),
                                       _ptr(workspace), workspace_bytes, _ptr(range_flag), kblock, flags),
           "emu_sgemm_batched_range")


def emu_sgemm_batched_host(m, n, k, alpha, A, lda, strideA, B, ldb, strideB, beta, C, ldc, strideC,
                           batch, mode, stream=None):
    _check(lib.emu_sgemm_batched_host(m, n, k, alpha, _ptr(A), lda, strideA, _ptr(B), ldb, strideB,
                                      beta, _ptr(C), ldc, strideC, batch, mode_of(mode), _stream(stream)),
           "emu_sgemm_batched_host")


def emu_sgemm(m, n, k, alpha, A, lda, B, ldb, beta, C, ldc, mode, stream=None):
    _check(lib.emu_sgemm(m, n, k, alpha, _ptr(A), lda, _ptr(B), ldb, beta, _ptr(C), ldc,
                         mode_of(mode), _stream(stream)), "emu_sgemm")


def emu_split(x, count, mode, hi, lo, stream=None):
    _check(lib.emu_split(_ptr(x), count, mode_of(mode), _ptr(hi), _ptr(lo), _stream(stream)), "emu_split")


def emu_tcec_gemm_batched(m, n, k, alpha, A, lda, strideA, B, ldb, strideB, beta, C, ldc, strideC,
                          batch, mode, stream=None, kblock=0, flags=0):
    _check(lib.emu_tcec_gemm_batched(m, n, k, alpha, _ptr(A), lda, strideA, _ptr(B), ldb, strideB,
                                     beta, _ptr(C), ldc, strideC, batch, mode_of(mode), _stream(stream),
                                     kblock, flags),
           "emu_tcec_gemm_batched")


def emu_tcec_householder_batched(m, n, V, strideV, X, ldx, strideX, C, ldc, strideC, batch, mode,
                                 stream=None, flags=0):
    _check(lib.emu_tcec_householder_batched(m, n, _ptr(V), strideV, _ptr(X), ldx, strideX, _ptr(C), ldc,
                                            strideC, batch, mode_of(mode), _stream(stream), flags),
           "emu_tcec_householder_batched")


def emu_tcec_givens_batched(m, n, i, j, CS, X, ldx, strideX, C, ldc, strideC, batch, mode, stream=None,
                            flags=0):
    _check(lib.emu_tcec_givens_batched(m, n, i, j, _ptr(CS), _ptr(X), ldx, strideX, _ptr(C), ldc, strideC,
                                       batch, mode_of(mode), _stream(stream), flags),
           "emu_tcec_givens_batched")


def emu_tcec_scan(n, count, X, ldx, Y, ldy, mode, stream=None, flags=0):
    _check(lib.emu_tcec_scan(n, count, _ptr(X), ldx, _ptr(Y), ldy, mode_of(mode), _stream(stream), flags),
           "emu_tcec_scan")


def emu_sgemm_batched_layout(layout, transa, transb, m, n, k, alpha, A, lda, strideA, B, ldb, strideB, beta, C,
                             ldc, strideC, batch, mode, stream=None, range_flag=None, kblock=0, flags=0):
    _check(lib.emu_sgemm_batched_layout(layout, transa.encode() if isinstance(transa, str) else transa,
                                        transb.encode() if isinstance(transb, str) else transb,
                                        m, n, k, alpha, _ptr(A), lda, strideA, _ptr(B), ldb, strideB,
                                        beta, _ptr(C), ldc, strideC, batch, mode_of(mode), _stream(stream),
                                        _ptr(range_flag), kblock, flags),
           "emu_sgemm_batched_layout")


def _rm_operand(x, name):
    """(trans, ld, batch stride) of a row-major 2-D / 3-D float32 CUDA tensor view:
    'N' when rows are contiguous, 'T' when columns are (a transposed view)."""
    import torch
    if x.dtype != torch.float32 or not x.is_cuda or x.dim() not in (2, 3):
        raise TypeError(f"{name}: a 2-D or 3-D float32 CUDA tensor is required")
    r, c = x.stride()[-2], x.stride()[-1]
    rows, cols = x.shape[-2], x.shape[-1]
    sb = x.stride()[0] if x.dim() == 3 else 0
    if c == 1 and r >= max(1, cols):
        return "N", r, sb
    if r == 1 and c >= max(1, rows):
        return "T", c, sb
    raise ValueError(f"{name}: rows or columns must be contiguous")


def matmul(A, B, mode="fp16", out=None, stream=None):
    """C = A @ B for float32 CUDA tensors (torch.matmul semantics for 2-D / 3-D
    operands; a 2-D operand is shared by every problem of a 3-D one), emulated by
    the library: one emu_sgemm_batched_layout call (row-major), nothing computed here."""
    import torch
    ta, lda, sA = _rm_operand(A, "A")
    tb, ldb, sB = _rm_operand(B, "B")
    m, k = A.shape[-2], A.shape[-1]
    k2, n = B.shape[-2], B.shape[-1]
    if k != k2:
        raise ValueError(f"inner dimensions differ: {k} vs {k2}")
    batch = A.shape[0] if A.dim() == 3 else (B.shape[0] if B.dim() == 3 else 1)
    if A.dim() == 3 and B.dim() == 3 and A.shape[0] != B.shape[0]:
        raise ValueError("batch sizes differ")
    shape = (batch, m, n) if (A.dim() == 3 or B.dim() == 3) else (m, n)
    if out is None:
        out = torch.empty(shape, dtype=torch.float32, device=A.device)
    elif tuple(out.shape) != shape or not out.is_contiguous():
        raise ValueError("out must be a contiguous tensor of the result shape")
    if out.numel() == 0:
        return out
    emu_sgemm_batched_layout(EMU_ROW_MAJOR, ta, tb, m, n, k, 1.0, A, lda, sA, B, ldb, sB, 0.0, out, max(1, n),
                             m * n, batch, mode, stream)
    return out


def emu_sgemm_multicast(m, n, k, alpha, A, lda, B, ldb, C_dst, ldc, mode, stream=None, kblock=0, flags=0):
    """C_dst: sequence of device buffers / addresses (1..8), each receiving C = alpha A B."""
    arr = (_p * len(C_dst))(*[_ptr(c) for c in C_dst])
    _check(lib.emu_sgemm_multicast(m, n, k, alpha, _ptr(A), lda, _ptr(B), ldb, arr, len(C_dst), ldc,
                                   mode_of(mode), _stream(stream), kblock, flags),
           "emu_sgemm_multicast")


def emu_status_string(status: int) -> str:
    return lib.emu_status_string(status).decode()


def emu_version() -> int:
    return lib.emu_version()


def emu_last_launch_count() -> int:
    return lib.emu_last_launch_count()


def emu_last_kernel_name() -> str:
    return lib.emu_last_kernel_name().decode()
