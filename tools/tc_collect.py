"""Collect tensor-core accumulation samples through the public C ABI (GPU box).

Operands exactly representable in FP16 / TF32 make the split's lo parts zero, so
D_corr = 0 and, for k <= KB, every output is the tensor core's own sum D_hi of
k exact products (one MMA instruction per K_inst = 16 FP16 / 8 TF32 products,
accumulating in TMEM between instructions).  General FP32 operands exercise the
whole path (P2/P3 interleaved in D_corr, the outside combine).  The samples are
written to gpurun_out/tc_samples.npz and fitted on the CPU by tools/tc_fit.py.

    python tools/tc_collect.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))

from gpu_util import emu_gpu  # noqa: E402


def representable(rng, shape, mode, emin, emax, pzero=0.05):
    """random values with 11 significant bits (FP16 normal range / TF32),
    random sign, exponent uniform in [emin, emax]"""
    sig = rng.integers(1024, 2048, size=shape).astype(np.float64)   # 11-bit significand
    e = rng.integers(emin, emax + 1, size=shape)
    x = np.ldexp(sig, e - 10) * rng.choice([-1.0, 1.0], size=shape)
    x[rng.random(shape) < pzero] = 0.0
    x = x.astype(np.float32)
    if mode == 0:
        assert np.all(x.astype(np.float16).astype(np.float32) == x)
    return x


def main():
    rng = np.random.default_rng(2308)
    out = {}
    cases = []
    for mode in (0, 1):
        for m in (128, 256):        # single-CTA kernel / CTA-pair TS kernel
            for k in (16, 32, 64):
                for (lo, hi) in ((-3, 3), (-12, 12), (-1, 0)):
                    cases.append(("rep", mode, m, 128, k, lo, hi, 0))
        for m in (128, 256):
            for k in (64, 256):
                cases.append(("gen", mode, m, 128, k, 0, 0, 0))
                cases.append(("gen", mode, m, 128, k, 0, 0, 128))
    for i, (kind, mode, m, n, k, lo, hi, kblock) in enumerate(cases):
        if kind == "rep":
            A = representable(rng, (k, m), mode, lo, hi)
            B = representable(rng, (n, k), mode, lo, hi)
        else:
            A = rng.uniform(-1, 1, size=(k, m)).astype(np.float32)
            B = rng.uniform(-1, 1, size=(n, k)).astype(np.float32)
        C = emu_gpu(mode, A, B, m, n, k, kblock=kblock)[0]
        tag = f"c{i}"
        out[tag + "_A"] = A
        out[tag + "_B"] = B
        out[tag + "_C"] = C
        out[tag + "_meta"] = np.array([mode, m, n, k, kblock, lo, hi, 1 if kind == "gen" else 0])
        print(tag, kind, mode, m, n, k, lo, hi, kblock, flush=True)
    os.makedirs("gpurun_out", exist_ok=True)
    np.savez_compressed("gpurun_out/tc_samples.npz", **out)
    print("saved", len(cases), "cases")


if __name__ == "__main__":
    main()
