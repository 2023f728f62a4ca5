"""Event trace of the leader CTA of cluster 0 (EMU_PROF build, tools/ only):
runs one c2 launch and prints the per-k-block timeline statistics of the TS
kernel -- where the MMA issuer, the splitters and the combine warps wait.

  python tools/trace.py [fp16|tf32] [batch | c3 | c3h]   (c3: one 16384^3 GEMM, c3h: 8192^3)
"""
import ctypes
import os
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import prof_roles  # noqa: E402

NAMES = {1: "prod_issue", 2: "spl_got_f32", 3: "spl_got_op", 4: "spl_done", 5: "mma_corr_start",
         6: "mma_corr_commit", 7: "mma_hi_start", 8: "mma_hi_commit", 9: "mma_got_op", 10: "epi_corr_full",
         11: "epi_corr_rel", 12: "epi_hi_full", 13: "epi_hi_rel", 14: "epi_store_start", 15: "epi_store_end",
         16: "epi_store_waited", 17: "epi_store_staged"}


def main():
    mode = 0 if (len(sys.argv) <= 1 or sys.argv[1] == "fp16") else 1
    shape = sys.argv[2] if len(sys.argv) > 2 else "1024"
    if shape in ("c3", "c3h"):
        batch, m = 1, (16384 if shape == "c3" else 8192)
    else:
        batch, m = int(shape), 256
    os.environ["EMU_EXTRA_DEFS"] = (os.environ.get("EMU_EXTRA_DEFS", "") + " -DEMU_TRACE").strip()
    prof_roles.build()
    L = ctypes.CDLL(prof_roles.LIB)
    n = k = m
    A = torch.rand(batch, k, m, device="cuda") * 2 - 1
    B = torch.rand(batch, n, k, device="cuda") * 2 - 1
    C = torch.empty(batch, n, m, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    P = ctypes.c_void_p
    L.emu_sgemm_batched.argtypes = [ctypes.c_int] * 3 + [ctypes.c_float, P, ctypes.c_int, ctypes.c_longlong, P,
                                    ctypes.c_int, ctypes.c_longlong, ctypes.c_float, P, ctypes.c_int,
                                    ctypes.c_longlong, ctypes.c_int, ctypes.c_int, P]
    call = lambda: L.emu_sgemm_batched(m, n, k, 1.0, A.data_ptr(), m, k * m, B.data_ptr(), k, n * k, 0.0,  # noqa
                                       C.data_ptr(), m, n * m, batch, mode, s)
    for _ in range(3):
        assert call() == 0
    torch.cuda.synchronize()
    L.emu_prof_reset()
    assert call() == 0
    torch.cuda.synchronize()
    R, NR = 1 << 12, 20
    buf = (ctypes.c_longlong * (2 * NR * R))()
    cnts = (ctypes.c_uint * NR)()
    assert L.emu_trace_read(buf, cnts) == NR
    print("trace counts per role:", list(cnts))
    allev = np.frombuffer(buf, dtype=np.int64).reshape(NR * R, 2).copy()
    for r in range(3, 19):   # combine warps: tag the warp in the high arg bits
        allev[r * R:r * R + cnts[r], 1] |= (r - 3) << 16
    # per-combine-warp release times of D_corr / D_hi, for the spread across warps
    rel = {}
    for r in range(3, 19):
        e_ = allev[r * R:r * R + cnts[r]]
        for code_ in (11, 13):
            rel.setdefault(code_, []).append(e_[(e_[:, 1] >> 32) == code_, 0])
    ev = np.concatenate([allev[r * R:r * R + cnts[r]] for r in range(3)] + [allev[3 * R:3 * R + cnts[3]]])
    cnt = len(ev)
    ev = ev[np.argsort(ev[:, 0], kind="stable")]
    for code_, name_ in ((11, "D_corr"), (13, "D_hi")):
        nmin = min(len(x) for x in rel[code_])
        if nmin == 0:
            print(name_, "release events per warp:", [len(x) for x in rel[code_]])
            continue
        M_ = np.stack([x[:nmin] for x in rel[code_]])
        spread = M_.max(0) - M_.min(0)
        last = np.argmax(M_, axis=0)
        print(f"release spread of {name_} over the 16 combine warps: mean {spread.mean():.0f} p50 "
              f"{np.median(spread):.0f} p90 {np.percentile(spread, 90):.0f} clk; last warp histogram "
              f"{np.bincount(last, minlength=16).tolist()}")
    t0 = ev[0, 0]
    t = ev[:, 0] - t0
    code = ev[:, 1] >> 32
    print(f"mode={mode} batch={batch} events={cnt} span={t[-1]} clk ({t[-1] / 1.9e3:.1f} us @1.9GHz)")
    # per event: sequence of times
    seq = defaultdict(list)
    for ti, c in zip(t, code):
        seq[int(c)].append(int(ti))
    for c in sorted(seq):
        print(f"  {NAMES.get(c, c):16s} n={len(seq[c])}")

    def pair_stats(a, b, label, shift=0):
        xa, xb = np.array(seq[a]), np.array(seq[b])
        nn = min(len(xa) - shift, len(xb))
        if nn <= 0:
            return
        d = xb[:nn] - xa[shift:shift + nn]
        print(f"  {label:44s} mean {d.mean():8.0f}  p50 {np.median(d):8.0f}  p90 {np.percentile(d, 90):8.0f} clk")

    print("intervals (clk):")
    pair_stats(5, 6, "MMA: corr issue (start -> commit)")
    pair_stats(6, 7, "MMA: wait D_hi free (corr commit -> hi start)")
    pair_stats(7, 8, "MMA: hi issue (start -> commit)")
    pair_stats(8, 5, "MMA: wait D_corr free (hi commit -> next corr)", shift=0) if False else None
    xa, xb = np.array(seq[8]), np.array(seq[5])
    if len(xb) > 1:
        d = xb[1:] - xa[:len(xb) - 1]
        print(f"  {'MMA: hi commit -> next corr start':44s} mean {d.mean():8.0f}  p50 {np.median(d):8.0f}  p90 {np.percentile(d, 90):8.0f} clk")
    x5 = np.array(seq[5])
    d = np.diff(x5)
    print(f"  {'MMA: k-block period (corr start -> next)':44s} mean {d.mean():8.0f}  p50 {np.median(d):8.0f}  p90 {np.percentile(d, 90):8.0f} clk")
    pair_stats(6, 10, "corr commit -> combine sees corr_full")
    pair_stats(10, 11, "combine: corr ld + release")
    pair_stats(8, 12, "hi commit -> combine sees hi_full")
    pair_stats(12, 13, "combine: hi ld + release")
    pair_stats(14, 15, "epilogue store")
    pair_stats(14, 16, "  store: wait previous bulk read")
    pair_stats(16, 17, "  store: stage 32 x 32 in smem + fence")
    pair_stats(17, 15, "  store: issue TMA store")
    pair_stats(3, 2, "splitter: got op slot -> got f32")
    pair_stats(2, 4, "splitter: split work")
    x4, x2 = np.array(seq[4]), np.array(seq[3])
    d = x2[1:] - x4[:len(x2) - 1]
    print(f"  {'splitter: done -> next op slot':44s} mean {d.mean():8.0f}  p50 {np.median(d):8.0f}  p90 {np.percentile(d, 90):8.0f} clk")
    d = np.diff(np.array(seq[4]))
    print(f"  {'splitter: stage period':44s} mean {d.mean():8.0f}  p50 {np.median(d):8.0f}  p90 {np.percentile(d, 90):8.0f} clk")
    d = np.diff(np.array(seq[1]))
    print(f"  {'producer: issue period':44s} mean {d.mean():8.0f}  p50 {np.median(d):8.0f}  p90 {np.percentile(d, 90):8.0f} clk")
    # first 140 events of a steady-state unit as a raw timeline
    mid = len(t) // 2
    print("raw timeline (steady state):")
    for i in range(mid, min(mid + 120, len(t))):
        print(f"  {t[i]:9d}  {NAMES.get(int(code[i]), code[i]):16s} {int(ev[i, 1] & 0xffffffff)}")


if __name__ == "__main__":
    main()
