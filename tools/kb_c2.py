"""c2 (1024 x 256^3) throughput vs the combine interval KB, both modes
(accuracy of each KB: tools/kb_accuracy.py, CPU)."""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2308_15152_b200 as emu  # noqa: E402

batch, N = 1024, 256
A = torch.rand(batch, N, N, device="cuda") * 2 - 1
B = torch.rand(batch, N, N, device="cuda") * 2 - 1
C = torch.empty(batch, N, N, device="cuda")
out = {}
for rep in range(2):
    for mode in ("fp16", "tf32"):
        for kb in (32, 64, 128, 256):
            f = lambda: emu.emu_sgemm_batched_ex(N, N, N, 1.0, A, N, N * N, B, N, N * N, 0.0, C, N, N * N, batch,
                                                 mode, None, None, kb, 0)
            for _ in range(5):
                f()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(50):
                f()
            b.record()
            torch.cuda.synchronize()
            ms = a.elapsed_time(b) / 50
            out[f"{mode}_kb{kb}_r{rep}"] = round(2.0 * batch * N ** 3 / ms / 1e9, 1)
print(json.dumps(out), flush=True)
