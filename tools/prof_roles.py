"""Role timing of the GEMM kernel: builds a -DEMU_PROF variant of the library
(tools/libemusgemm_prof.so, never used by the product), runs one workload and
prints where each warp role spends its cycles.

  python tools/prof_roles.py [c2|c3] [fp16|tf32] [reps]
"""
import ctypes
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2308_15152_b200 import build as B  # noqa: E402

LIB = os.path.join(ROOT, "tools", "libemusgemm_prof.so")
SLOTS = ["prod_wait_empty", "mma_wait_acc", "mma_wait_op", "spl_wait_f32", "spl_wait_op", "spl_work",
         "epi_wait_acc", "epi_drain", "epi_store", "cta_total", "mma_issue"]


def build():
    flags = list(B.FLAGS)
    i = flags.index("-Xptxas")
    del flags[i:i + 2]
    extra = os.environ.get("EMU_EXTRA_DEFS", "").split()   # e.g. -DEMU_TS_MMA_WARP=3 (experiments)
    cmd = [B.NVCC, *flags, "-DEMU_PROF", *extra, "-o", LIB, *B.SOURCES]
    subprocess.check_call(cmd, stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
    mode = 0 if (len(sys.argv) <= 2 or sys.argv[2] == "fp16") else 1
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
    build()
    L = ctypes.CDLL(LIB)
    if cfg == "c2":
        batch, m, n, k = 1024, 256, 256, 256
    elif cfg == "c3h":
        batch, m, n, k = 1, 8192, 8192, 8192
    else:
        batch, m, n, k = 1, 16384, 16384, 16384
    A = torch.rand(batch, k, m, device="cuda") * 2 - 1
    Bm = torch.rand(batch, n, k, device="cuda") * 2 - 1
    C = torch.empty(batch, n, m, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    P = ctypes.c_void_p
    L.emu_sgemm_batched.argtypes = [ctypes.c_int] * 3 + [ctypes.c_float, P, ctypes.c_int, ctypes.c_longlong, P,
                                    ctypes.c_int, ctypes.c_longlong, ctypes.c_float, P, ctypes.c_int,
                                    ctypes.c_longlong, ctypes.c_int, ctypes.c_int, P]
    call = lambda: L.emu_sgemm_batched(m, n, k, 1.0, A.data_ptr(), m, k * m, Bm.data_ptr(), k, n * k, 0.0,  # noqa
                                       C.data_ptr(), m, n * m, batch, mode, s)
    assert call() == 0
    torch.cuda.synchronize()
    L.emu_prof_reset()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for _ in range(reps):
        assert call() == 0
    ev1.record()
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / reps
    buf = (ctypes.c_ulonglong * 16)()
    L.emu_prof_read(buf, 16)
    v = {k_: buf[i] for i, k_ in enumerate(SLOTS)}
    ctas = 148 * reps
    tot = v["cta_total"] / ctas
    print(f"{cfg} mode={mode} {ms:.3f} ms/launch, {2.0 * m * n * k * batch / ms / 1e9:.1f} TF; "
          f"cycles per CTA {tot:.0f}")
    kern = os.environ.get("EMU_KERNEL", "ts")
    nspl = 8 if kern in ("single", "ts") or m <= 128 else 16
    nepi = 16 if kern == "ts" and m > 128 else 8
    ctas_mma = ctas if (kern == "single" or m <= 128) else ctas // 2   # pair kernels: the MMA issuer lives in the leader CTA
    per = {"prod_wait_empty": 1, "mma_wait_acc": ctas_mma / ctas, "mma_wait_op": ctas_mma / ctas,
           "mma_issue": ctas_mma / ctas, "spl_wait_f32": nspl, "spl_wait_op": nspl, "spl_work": nspl,
           "epi_wait_acc": nepi, "epi_drain": nepi, "epi_store": nepi}
    for k_, nw in per.items():
        print(f"  {k_:16s} {v[k_] / ctas / nw / tot * 100:6.1f}% of CTA time (per warp)")


if __name__ == "__main__":
    main()
