"""GPU split parity: emu_split (the device code the GEMM's splitter warps run)
is bit-exact with the oracle's split (Eqs. corr-1..corr-4; R#6 for
TF32) on all 2^32 binary32 inputs; NaNs compare by NaN-ness."""
import concurrent.futures
import os

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu
CHUNK = 1 << 26


def _run(mode):
    import torch
    import paper_2308_15152_b200 as emu
    x = torch.empty(CHUNK, dtype=torch.int64, device="cuda")
    hi = torch.empty(CHUNK, dtype=torch.int16 if mode == "fp16" else torch.int32, device="cuda")
    lo = torch.empty_like(hi)
    nthr = max(1, min(32, os.cpu_count() or 1))
    oracle.set_threads(nthr)

    def cpu_ref(c):
        u = np.arange(c, c + CHUNK, dtype=np.uint64).astype(np.uint32)
        if mode == "fp16":
            h, l = oracle.split_fp16(u.view(np.float32))
            return h.view(np.int16), l.view(np.int16), u
        h, l = oracle.split_tf32(u.view(np.float32))
        return h.view(np.int32), l.view(np.int32), u

    bad = 0
    with concurrent.futures.ThreadPoolExecutor(1) as ex:
        fut = ex.submit(cpu_ref, 0)
        for c in range(0, 1 << 32, CHUNK):
            torch.arange(c, c + CHUNK, dtype=torch.int64, device="cuda", out=x)
            xf = x.to(torch.int32).view(torch.float32)   # wraps to the same 32-bit patterns
            emu.emu_split(xf, CHUNK, mode, hi, lo)
            gh, gl = hi.cpu().numpy(), lo.cpu().numpy()
            rh, rl, u = fut.result()
            if c + CHUNK < (1 << 32):
                fut = ex.submit(cpu_ref, c + CHUNK)
            xv = u.view(np.float32)
            nan_in = np.isnan(xv)
            if mode == "fp16":
                fin = ~nan_in
                bad += int(np.count_nonzero((gh != rh) & fin))
                # lo of finite inputs; for NaN inputs both parts must be NaN
                rnan = ((rl.view(np.uint16) & 0x7c00) == 0x7c00) & ((rl.view(np.uint16) & 0x3ff) != 0)
                gnan_l = ((gl.view(np.uint16) & 0x7c00) == 0x7c00) & ((gl.view(np.uint16) & 0x3ff) != 0)
                bad += int(np.count_nonzero((gl != rl) & fin & ~(rnan & gnan_l)))
                gnan = ((gh.view(np.uint16) & 0x7c00) == 0x7c00) & ((gh.view(np.uint16) & 0x3ff) != 0)
                bad += int(np.count_nonzero(nan_in & ~gnan))
            else:
                fin = ~nan_in
                same = (gh == rh) & ((gl == rl) | (np.isnan(gl.view(np.float32)) & np.isnan(rl.view(np.float32))))
                bad += int(np.count_nonzero(~same & fin))
                bad += int(np.count_nonzero(nan_in & ~np.isnan(gh.view(np.float32))))
            if bad:
                i = int(np.argmax(((gh != rh) | (gl != rl)) & fin))
                raise AssertionError(f"mode {mode}: input {hex(int(u[i]))}: gpu ({hex(int(gh[i]))}, "
                                     f"{hex(int(gl[i]))}) oracle ({hex(int(rh[i]))}, {hex(int(rl[i]))})")
    return bad


@pytest.mark.parametrize("mode", ["fp16", "tf32"])
def test_split_bit_exact_all_inputs(mode):
    assert _run(mode) == 0
