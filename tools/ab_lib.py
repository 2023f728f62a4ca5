"""Interleaved A/B of two builds of libemusgemm.so on c2 (1024 x 256^3) and c3
(16384^3): the same inputs and launch, alternating libraries, CUDA-event timing.

    python tools/ab_lib.py LIB_A.so LIB_B.so [LIB_C.so ...] [rounds] [kblock]
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


def clocks():
    try:
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(0)
        return (pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                round(pynvml.nvmlDeviceGetPowerUsage(h) / 1000))
    except Exception:
        return (None, None)


def main():
    paths = [a for a in sys.argv[1:] if a.endswith(".so")]
    rest = [a for a in sys.argv[1:] if not a.endswith(".so")]
    names = [chr(ord("A") + i) for i in range(len(paths))]
    libs = {nm: load(pth) for nm, pth in zip(names, paths)}
    rounds = int(rest[0]) if len(rest) > 0 else 3
    kb = int(rest[1]) if len(rest) > 1 else 64
    res = {}
    # ABBA order per round so that drift over time favours neither library
    for shape, (batch, N, it) in {"c2": (1024, 256, 1000), "c3": (1, 16384, 5)}.items():
        A = torch.rand(batch, N, N, device="cuda") * 2 - 1
        B = torch.rand(batch, N, N, device="cuda") * 2 - 1
        C = torch.empty(batch, N, N, device="cuda")
        for r in range(rounds):
            for mode in (0, 1):
                for name in names + names[::-1]:
                    key = f"{shape}_{'fp16' if mode == 0 else 'tf32'}_{name}"
                    tf = round(timed(libs[name], batch, N, A, B, C, mode, kb, it), 1)
                    res.setdefault(key, []).append(tf)
                    res.setdefault(key + "_clk_pow", []).append(clocks())
        del A, B, C
        torch.cuda.empty_cache()
    summary = {k: round(sum(v) / len(v), 1) for k, v in res.items() if not k.endswith("_clk_pow")}
    print(json.dumps({"libs": dict(zip(names, paths)), "mean": summary, "all": res}), flush=True)


if __name__ == "__main__":
    main()
