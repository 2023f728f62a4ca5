"""Accuracy of the emulated GEMM vs the outside-combine interval KB, computed
with the oracle's measured tensor-core model (tc="sm100", R#9) --
no GPU needed: the model is bit-exact with the kernels.

For each k, a 64 x 64 block of outputs (64 random rows of A, 64 random columns
of B, uniform[-1,1]) is computed by the model at KB in {32, ..., 1024} and by
plain FP32 SGEMM (O5, sequential FMA); rel-Frobenius vs FP64 is reported as the
ratio to SGEMM's (north_star gate: <= 2).

    python tools/kb_accuracy.py [k ...]
"""
import sys

import numpy as np

sys.path.insert(0, ".")
import oracle      # noqa: E402
import workloads   # noqa: E402


def main():
    ks = [int(a) for a in sys.argv[1:]] or [256, 1024, 4096, 16384]
    m = n = 64
    print("mode k KB rel_frob(emu) rel_frob(sgemm) ratio")
    for mode in ("fp16", "tf32"):
        for k in ks:
            A = workloads.uniform((1, k, m), seed=k)
            B = workloads.uniform((1, n, k), seed=k + 1)
            R = oracle.gemm_f64(A, B, m, n, k)
            es = oracle.rel_frobenius(oracle.sgemm_f32(A, B, m, n, k), R)
            for kb in (32, 64, 128, 256, 512, 1024):
                if kb > max(k, 64):
                    break
                C = oracle.emu_gemm(mode, A, B, m, n, k, kb=kb, tc="sm100")
                e = oracle.rel_frobenius(C, R)
                print(mode, k, kb, f"{e:.3e}", f"{es:.3e}", f"{e / es:.2f}", flush=True)


if __name__ == "__main__":
    main()
