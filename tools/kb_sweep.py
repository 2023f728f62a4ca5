"""Combine interval KB (R#7: tuned only upward within accuracy): c3-size
throughput and accuracy (rel-Frobenius vs FP64 against plain FP32 SGEMM) at
KB = 64 / 128 / 256, both modes."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import oracle  # noqa: E402
import paper_2308_15152_b200 as emu  # noqa: E402
import workloads  # noqa: E402


def t_ms(fn, it):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(it):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / it


out = {}
N = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
A = torch.rand(N, N, device="cuda") * 2 - 1
B = torch.rand(N, N, device="cuda") * 2 - 1
C = torch.empty(N, N, device="cuda")
for mode in ("fp16", "tf32"):
    for kb in (64, 128, 256):
        ms = t_ms(lambda: emu.emu_sgemm_batched_ex(N, N, N, 1.0, A, N, 0, B, N, 0, 0.0, C, N, 0, 1, mode, None,
                                                   None, kb, 0), 5)
        out[f"{mode}_kb{kb}_TF"] = round(2.0 * N ** 3 / ms / 1e9, 1)
print(json.dumps(out), flush=True)
# accuracy: 256 x 256 x k, uniform, 3 seeds (references computed once per problem)
for k in (1024, 4096):
    for seed in (1, 2, 3):
        Ah, Bh = workloads.make_operands(1, 256, 256, k, seed)
        R = oracle.gemm_f64(Ah, Bh, 256, 256, k)
        es = oracle.rel_frobenius(oracle.sgemm_f32(Ah, Bh, 256, 256, k), R)
        dA, dB = torch.from_numpy(Ah).cuda(), torch.from_numpy(Bh).cuda()
        for mode in ("fp16", "tf32"):
            for kb in (64, 128, 256):
                dC = torch.empty(1, 256, 256, device="cuda")
                emu.emu_sgemm_batched_ex(256, 256, k, 1.0, dA, 256, 0, dB, k, 0, 0.0, dC, 256, 0, 1, mode, None,
                                         None, kb, 0)
                e = oracle.rel_frobenius(dC.cpu().numpy(), R)
                key = f"acc_{mode}_k{k}_kb{kb}_ratio_to_sgemm"
                out[key] = round(max(out.get(key, 0.0), e / es), 3)
    print(json.dumps(out), flush=True)
