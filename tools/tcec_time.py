"""Time the device-API kernels (include/emu_tcec.cuh users) beside the library's
persistent kernel: c2 (1024 x 256^3) through emu_tcec_gemm_batched for every
policy, and the structured-operand kernels on batched shapes of the paper's
primitive benchmarks.  CUDA events, warm-up 3, median of 20."""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2308_15152_b200 as emu  # noqa: E402


def t_ms(fn, it=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(it):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2]


out = {}
batch, m = 1024, 256
A = torch.rand(batch, m, m, device="cuda") * 2 - 1
B = torch.rand(batch, m, m, device="cuda") * 2 - 1
C = torch.empty(batch, m, m, device="cuda")
fl = 2.0 * batch * m ** 3
for mode in ("fp16", "tf32"):
    ms = t_ms(lambda: emu.emu_sgemm_batched(m, m, m, 1.0, A, m, m * m, B, m, m * m, 0.0, C, m, m * m, batch, mode))
    out[f"c2_{mode}_library"] = round(fl / ms / 1e9, 1)
    for flags, name in ((0, "tc"), (1, "tc_noec"), (2, "simt"), (4, "pipelined"), (5, "pipelined_noec")):
        ms = t_ms(lambda: emu.emu_tcec_gemm_batched(m, m, m, 1.0, A, m, m * m, B, m, m * m, 0.0, C, m, m * m,
                                                    batch, mode, None, 0, flags), it=5 if flags & 2 else 20)
        out[f"c2_{mode}_tcec_{name}"] = round(fl / ms / 1e9, 1)
# structured: batched Householder / Givens on m x m reflectors times m x 128 blocks, scan
for hm in (32, 128, 256):
    nb, n = 4096, 128
    V = torch.nn.functional.normalize(torch.rand(nb, hm, device="cuda") - 0.5, dim=1)
    X = torch.rand(nb, n, hm, device="cuda")
    Y = torch.empty_like(X)
    ms = t_ms(lambda: emu.emu_tcec_householder_batched(hm, n, V, hm, X, hm, n * hm, Y, hm, n * hm, nb, "fp16"))
    out[f"householder_m{hm}_fp16_TFs"] = round(2.0 * nb * hm * hm * n / ms / 1e9, 1)
    ms = t_ms(lambda: emu.emu_tcec_householder_batched(hm, n, V, hm, X, hm, n * hm, Y, hm, n * hm, nb, "fp16",
                                                       None, 4))
    out[f"householder_m{hm}_fp16_pipelined_TFs"] = round(2.0 * nb * hm * hm * n / ms / 1e9, 1)
    CS = torch.rand(nb, 2, device="cuda")
    ms = t_ms(lambda: emu.emu_tcec_givens_batched(hm, n, 1, hm - 2, CS, X, hm, n * hm, Y, hm, n * hm, nb, "fp16"))
    out[f"givens_m{hm}_fp16_TFs"] = round(2.0 * nb * hm * hm * n / ms / 1e9, 1)
Xs = torch.rand(1 << 16, 1024, device="cuda")
Ys = torch.empty_like(Xs)
ms = t_ms(lambda: emu.emu_tcec_scan(1024, 1 << 16, Xs, 1024, Ys, 1024, "fp16"))
out["scan_1024x65536_fp16_GBs"] = round(2 * Xs.numel() * 4 / ms / 1e6, 1)
print(json.dumps(out))
