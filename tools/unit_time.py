"""Per-unit time of the c2-shaped batched GEMM vs batch size: small batches are
(nearly) L2-resident, so the time per (item, 256-row) unit there is the compute
pipeline's own pace; at 1024 it is the HBM-fed pace."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2308_15152_b200 as emu  # noqa: E402

m = n = k = 256
for mode in ("fp16", "tf32"):
    for batch in (148, 296, 592, 1024):
        A = torch.rand(batch, k, m, device="cuda") * 2 - 1
        B = torch.rand(batch, n, k, device="cuda") * 2 - 1
        C = torch.empty(batch, n, m, device="cuda")
        f = lambda: emu.emu_sgemm_batched(m, n, k, 1.0, A, m, k * m, B, k, n * k, 0.0, C, m, n * m, batch, mode)  # noqa
        for _ in range(5):
            f()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        reps = 50
        for _ in range(reps):
            f()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        units_per_cluster = batch / 74
        print(json.dumps({"mode": mode, "batch": batch, "ms": round(ms, 4),
                          "us_per_unit": round(ms * 1e3 / units_per_cluster, 3),
                          "TF": round(2 * m * n * k * batch / ms / 1e9, 1),
                          "GBs": round(3 * 4 * m * n * batch / ms / 1e6, 1)}), flush=True)
