"""Build libemusgemm.so in-tree for sm_100a with nvcc (no JIT cache: the .so
travels to the GPU box with the repo snapshot)."""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
SRC_DIR = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libemusgemm.so")
SOURCES = [os.path.join(SRC_DIR, "api.cu")]
DEPS = SOURCES + [os.path.join(SRC_DIR, f) for f in os.listdir(SRC_DIR) if f.endswith(".cuh")] + \
    [os.path.join(ROOT, "include", f) for f in os.listdir(os.path.join(ROOT, "include"))]

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden", "-shared",
         "-I", os.path.join(ROOT, "include"), "-I", SRC_DIR,
         "-Xptxas", "-v", "--expt-relaxed-constexpr"]


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(d) > t for d in DEPS)


def build(force: bool = False, verbose: bool = False) -> str:
    if force or stale():
        # EMU_BUILD_DEFS: extra -D flags for tuning experiments (tools/gpu_defab.sh)
        cmd = [NVCC, *FLAGS, *os.environ.get("EMU_BUILD_DEFS", "").split(), "-o", LIB, *SOURCES]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("nvcc failed building libemusgemm.so")
        if verbose:
            sys.stderr.write(r.stderr)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
