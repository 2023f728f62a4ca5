"""Standalone tcgen05 accumulator probe -- HARDWARE MEASUREMENT, test
infrastructure (see probe/tc_probe.cu for what it measures and why).

It shares no code with the product library (paper_2308_15152_b200) or with
the oracle: tests/test_gpu_tcprobe.py compares its outputs with the oracle's
instruction-level tensor-core model (oracle.tc_chain), and tools/tc_fit.py fits
that model's parameters to its samples only (R#9).

    run(kind, pair, a_tmem, A, B, D0=None) -> D
      kind "fp16" | "tf32"; pair: cta_group::2 (M = 256) instead of ::1 (M = 128);
      a_tmem: A operand from tensor memory instead of shared memory;
      A (grid, n, M, K_inst), B (grid, n, N, K_inst) exact operand VALUES
      (float32 arrays holding binary16 / TF32 values; converted to bit patterns
      here); D0 (grid, M, N) float32 or None.  Returns D (grid, M, N) float32.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "tc_probe.cu")
_LIB = os.path.join(_HERE, "libtcprobe.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
BUILD_CMD = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-O2", "-lineinfo", "-std=c++17",
             "-Xcompiler", "-fPIC", "-shared", "-o", _LIB, _SRC]
KINST = {"fp16": 16, "tf32": 8}


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(BUILD_CMD)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB):
            raise RuntimeError("probe/libtcprobe.so is missing: run __graft_entry__.build()")
        L = ctypes.CDLL(_LIB)
        i32, P = ctypes.c_int, ctypes.c_void_p
        L.tcp_run.argtypes = [i32, i32, i32, i32, i32, i32, P, P, P, P, P]
        L.tcp_run.restype = i32
        _lib = L
    return _lib


def operand_bits(kind: str, x) -> np.ndarray:
    """bit patterns of exact binary16 / TF32 values (asserts exactness)"""
    x = np.ascontiguousarray(x, dtype=np.float32)
    if kind == "fp16":
        h = x.astype(np.float16)
        assert np.array_equal(h.astype(np.float32), x), "operand not exact in binary16"
        return h.view(np.uint16)
    b = x.view(np.uint32)
    assert not np.any(b & 0x1FFF), "operand not exact in TF32"
    return b.copy()


def run(kind, pair, a_tmem, A, B, D0=None):
    import torch
    kind_i = {"fp16": 0, "tf32": 1}[kind]
    A = np.asarray(A, dtype=np.float32)
    B = np.asarray(B, dtype=np.float32)
    grid, n, M, K = A.shape
    N = B.shape[2]
    assert K == KINST[kind] and B.shape == (grid, n, N, K) and M == (256 if pair else 128)
    dA = torch.from_numpy(operand_bits(kind, A).view(np.uint8).copy()).cuda()
    dB = torch.from_numpy(operand_bits(kind, B).view(np.uint8).copy()).cuda()
    dD = torch.full((grid, M, N), float("nan"), device="cuda")
    dD0 = None if D0 is None else torch.from_numpy(np.ascontiguousarray(D0, dtype=np.float32)).cuda()
    rc = lib().tcp_run(kind_i, int(bool(pair)), int(bool(a_tmem)), n, N, grid, dA.data_ptr(), dB.data_ptr(),
                       None if dD0 is None else dD0.data_ptr(), dD.data_ptr(),
                       torch.cuda.current_stream().cuda_stream)
    if rc != 0:
        raise RuntimeError(f"tcp_run failed: {rc}")
    torch.cuda.synchronize()
    return dD.cpu().numpy()
