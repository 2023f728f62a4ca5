"""Small calls through every kernel the dispatch picks, for compute-sanitizer
(memcheck): single-CTA, direct-load, TS streaming / A-stationary / 64-wide,
range-safe, transposes, multicast, the device-API kernels."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import paper_2308_15152_b200 as emu  # noqa: E402
import workloads  # noqa: E402
from gpu_util import emu_gpu, emu_gpu_range  # noqa: E402

for mode in ("fp16", "tf32"):
    for (batch, m, n, k) in [(2, 100, 70, 90), (1, 300, 200, 300), (160, 256, 256, 256), (3, 257, 129, 77)]:
        A, B = workloads.make_operands(batch, m, n, k, seed=1)
        emu_gpu(mode, A, B, m, n, k)
    A, B = workloads.make_operands(1, 63, 61, 77, seed=2, lda=65, ldb=78)
    emu_gpu(mode, A, B, 63, 61, 77)
    A, B = workloads.make_operands(1, 256, 192, 300, seed=3, dist="logu30")
    emu_gpu_range(mode, A, B, 256, 192, 300)
    A, B = workloads.make_operands(2, 200, 136, 300, seed=4)
    dA = torch.from_numpy(np.ascontiguousarray(np.transpose(A, (0, 2, 1)))).cuda()
    dC = torch.empty((2, 136, 200), device="cuda")
    emu.emu_sgemm_batched_t("T", "N", 200, 136, 300, 1.0, dA, 300, 300 * 200, torch.from_numpy(B).cuda(), 300,
                            136 * 300, 0.0, dC, 200, 136 * 200, 2, mode)
    x = torch.rand(3, 128, 96, device="cuda")
    y = torch.rand(3, 80, 128, device="cuda")
    z = torch.empty(3, 80, 96, device="cuda")
    emu.emu_tcec_gemm_batched(96, 80, 128, 1.0, x, 96, 128 * 96, y, 128, 80 * 128, 0.0, z, 96, 80 * 96, 3, mode,
                              None, 0, 0)
torch.cuda.synchronize()
print("sanitize run ok")
