"""c4-shape timing breakdown: plain GEMM (64-wide few-tile path) vs the
range-safe entry (max-|x| pass + GEMM), and the tile-width choice."""
import json
import os
import sys

import torch

sys.path.insert(0, ".")
import paper_2308_15152_b200 as emu  # noqa: E402

m = n = 1024
k = 4096
A = torch.rand(k, m, device="cuda") * 2 - 1
B = torch.rand(n, k, device="cuda") * 2 - 1
C = torch.empty(n, m, device="cuda")
ws = torch.empty((m + n) * 4, dtype=torch.uint8, device="cuda")


def t(fn, it=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(it):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / it * 1e3


out = {}
for mode in ("fp16", "tf32"):
    us = t(lambda: emu.emu_sgemm_batched(m, n, k, 1.0, A, m, 0, B, k, 0, 0.0, C, m, 0, 1, mode))
    out[f"{mode}_plain_us"] = round(us, 1)
    out[f"{mode}_plain_TF"] = round(2 * m * n * k / us / 1e6, 1)
    us = t(lambda: emu.emu_sgemm_batched_range(m, n, k, 1.0, A, m, 0, B, k, 0, 0.0, C, m, 0, 1, mode, ws,
                                               ws.numel(), None, None, 0, 0))
    out[f"{mode}_range_us"] = round(us, 1)
# the same GEMM on operands scaled by 2^14 (the range-safe mode's operand magnitudes)
A2, B2 = A * 16384.0, B * 16384.0
for mode in ("fp16", "tf32"):
    us = t(lambda: emu.emu_sgemm_batched(m, n, k, 1.0, A2, m, 0, B2, k, 0, 0.0, C, m, 0, 1, mode))
    out[f"{mode}_plain_scaled_inputs_us"] = round(us, 1)
out["EMU_TS_N"] = os.environ.get("EMU_TS_N", "auto")
print(json.dumps(out))
