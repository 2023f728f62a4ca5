"""HBM ceilings for the c2 traffic pattern (read A and B, write C; 2:1 read:write)
measured with plain torch kernels: C = A + B on 268 MB tensors, a copy, a pure read.
Prints one JSON line per probe (GB/s counted as bytes read + written)."""
import json

import torch

n = 1024 * 256 * 256
a = torch.rand(n, device="cuda")
b = torch.rand(n, device="cuda")
c = torch.empty(n, device="cuda")
s = torch.empty(1, device="cuda")


def t(fn, reps=50):
    for _ in range(5):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(5):
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / reps)
    return best


for name, fn, byts in [("add_2r1w", lambda: torch.add(a, b, out=c), 12 * n),
                       ("copy_1r1w", lambda: c.copy_(a), 8 * n),
                       ("sum_1r", lambda: torch.sum(a, dim=0, out=s[0]), 4 * n)]:
    ms = t(fn)
    print(json.dumps({"probe": name, "ms": round(ms, 4), "GBs": round(byts / ms / 1e6, 1)}))
