"""Quick GPU sanity run: small GEMMs through the C ABI vs the oracle, printing
error statistics instead of asserting (first-contact debugging)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
import workloads  # noqa: E402
from gpu_util import emu_gpu, tolerance  # noqa: E402

for mode in ("fp16", "tf32"):
    for (batch, m, n, k) in [(150, 200, 300, 96), (1, 128, 128, 32), (1, 128, 128, 64), (1, 128, 128, 256), (2, 200, 136, 300), (1, 256, 128, 64), (3, 300, 260, 200),
                             (16, 64, 64, 64)]:
        A, B = workloads.make_operands(batch, m, n, k, seed=1)
        try:
            C = emu_gpu(mode, A, B, m, n, k)
        except Exception as e:  # noqa: BLE001
            print(mode, (batch, m, n, k), "ERROR", e, flush=True)
            continue
        ref = oracle.emu_gemm(mode, A, B, m, n, k)
        tol = tolerance(mode, A, B, m, n, k)
        d = np.abs(C.astype(np.float64) - ref)
        bad = ~(d <= tol)
        R = oracle.gemm_f64(A, B, m, n, k)
        print(mode, (batch, m, n, k), "nan:", int(np.isnan(C).sum()), "bad:", int(bad.sum()), "of", C.size,
              "max d/tol: %.3g" % np.nanmax(d / tol), "relF: %.3g" % oracle.rel_frobenius(np.nan_to_num(C), R),
              flush=True)
        if bad.any():
            b, j, i = np.argwhere(bad)[0]
            print("   first bad (b,i,j)=", (b, i, j), "gpu", C[b, j, i], "ref", ref[b, j, i], flush=True)
            # pattern of bad rows / cols
            print("   bad rows:", np.unique(np.argwhere(bad)[:, 2])[:20], " bad cols:",
                  np.unique(np.argwhere(bad)[:, 1])[:20], flush=True)
