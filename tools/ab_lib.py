"""Interleaved A/B of two builds of libemusgemm.so on c2 (1024 x 256^3) and c3
(16384^3): the same inputs and launch, alternating libraries, CUDA-event timing.

    python tools/ab_lib.py LIB_A LIB_B [rounds]
"""
import ctypes
import json
import sys

import torch


def load(path):
    L = ctypes.CDLL(path)
    i, ll, f, p = ctypes.c_int, ctypes.c_longlong, ctypes.c_float, ctypes.c_void_p
    L.emu_sgemm_batched_ex.argtypes = [i, i, i, f, p, i, ll, p, i, ll, f, p, i, ll, i, i, p, p, i, ctypes.c_uint]
    L.emu_sgemm_batched_ex.restype = i
    return L


def timed(L, batch, N, A, B, C, mode, kb, it):
    s = torch.cuda.current_stream().cuda_stream

    def f():
        rc = L.emu_sgemm_batched_ex(N, N, N, 1.0, A.data_ptr(), N, N * N, B.data_ptr(), N, N * N, 0.0,
                                    C.data_ptr(), N, N * N, batch, mode, s, None, kb, 0)
        assert rc == 0, rc
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(it):
        f()
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / it
    return 2.0 * batch * N ** 3 / ms / 1e9


def main():
    libs = {"A": load(sys.argv[1]), "B": load(sys.argv[2])}
    rounds = int(sys.argv[3]) if len(sys.argv) > 3 else 3
    res = {}
    for shape, (batch, N, it) in {"c2": (1024, 256, 100), "c3": (1, 16384, 3)}.items():
        A = torch.rand(batch, N, N, device="cuda") * 2 - 1
        B = torch.rand(batch, N, N, device="cuda") * 2 - 1
        C = torch.empty(batch, N, N, device="cuda")
        for r in range(rounds):
            for mode in (0, 1):
                if shape == "c3" and mode == 1 and r > 0:
                    continue
                for name, L in libs.items():
                    key = f"{shape}_{'fp16' if mode == 0 else 'tf32'}_{name}"
                    res.setdefault(key, []).append(round(timed(L, batch, N, A, B, C, mode, 64, it), 1))
        del A, B, C
        torch.cuda.empty_cache()
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
