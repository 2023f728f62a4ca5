"""GPU-side helpers for the parity tests: run the C ABI on column-major numpy
operands (layout of `workloads`) and compute the element-wise tolerance
 from the oracle's |A||B|."""
import math

import numpy as np

import oracle

U = 2.0 ** -24


def emu_gpu(mode, A, B, m, n, k, alpha=1.0, beta=0.0, C=None, kblock=0, flags=0, range_flag=None,
            ldc=None):
    import torch
    import paper_2308_15152_b200 as emu
    A = np.ascontiguousarray(A, dtype=np.float32)
    B = np.ascontiguousarray(B, dtype=np.float32)
    if A.ndim == 2:
        A = A[None]
    if B.ndim == 2:
        B = B[None]
    batch = max(A.shape[0], B.shape[0])
    lda, ldb = A.shape[2], B.shape[2]
    sA = 0 if (A.shape[0] == 1 and batch > 1) else A.shape[1] * lda
    sB = 0 if (B.shape[0] == 1 and batch > 1) else B.shape[1] * ldb
    ldc = m if ldc is None else ldc
    dA = torch.from_numpy(A).cuda()
    dB = torch.from_numpy(B).cuda()
    if C is None:
        dC = torch.full((batch, n, ldc), float("nan"), device="cuda")
    else:
        dC = torch.from_numpy(np.ascontiguousarray(C, dtype=np.float32).reshape(batch, n, ldc)).cuda()
    emu.emu_sgemm_batched_ex(m, n, k, alpha, dA, lda, sA, dB, ldb, sB, beta, dC, ldc, n * ldc, batch,
                             mode, None, range_flag, kblock, flags)
    torch.cuda.synchronize()
    return dC.cpu().numpy()


def assert_bits_equal(got, want):
    """element-wise equality by value (-0 == +0; NaN == NaN), with a readable
    report of the first mismatches"""
    got = np.asarray(got, dtype=np.float32)
    want = np.asarray(want, dtype=np.float32)
    assert got.shape == want.shape, (got.shape, want.shape)
    bad = ~((got == want) | (np.isnan(got) & np.isnan(want)))
    if np.any(bad):
        idx = np.argwhere(bad)[:5]
        rows = [(tuple(int(v) for v in ix), float(got[tuple(ix)]), float(want[tuple(ix)])) for ix in idx]
        raise AssertionError(f"{int(bad.sum())} of {bad.size} outputs differ from the oracle: {rows}")


def tolerance_abab(mode, A, B, m, n, k, kblock=0):
    """The round-1 bar (kept for the device-API tests, which scale it):
        gamma = 2*(KB/K_inst) + 4 + 2*ceil(k/KB),  tol = gamma * u * (|A||B|)_ij
    Loose at large k (its cross-block term grows with |A||B|, not |C|)."""
    kb = kblock or oracle.default_kb(k)
    kinst = 16 if mode in (0, "fp16") else 8
    gamma = 2 * (kb / kinst) + 4 + 2 * math.ceil(max(k, 1) / kb)
    A = np.asarray(A)
    B = np.asarray(B)
    if A.ndim == 2:
        A = A[None]
    if B.ndim == 2:
        B = B[None]
    batch = max(A.shape[0], B.shape[0])
    out = np.empty((batch, n, m))
    for b in range(batch):
        out[b] = oracle.absgemm_f64(A[b if A.shape[0] > 1 else 0], B[b if B.shape[0] > 1 else 0], m, n, k)
    return gamma * U * out


JMIN_GRID = 2.0 ** -158     # the adder's lowest alignment bit (R#9)


def entry_bound(mode, a, b, kb, corr=True):
    """Rigorous (first-order, 2 % slack) bound on |C_gpu - C_oracle("ideal")|
    for outputs C = sum_p a[e, p] b[e, p] (a, b: (E, k) operand values), alpha = 1,
    beta = 0.  Both sides use the same split (bit-exact, R#1-6) and the same
    exact products; they differ only in how each k-block's sums are formed:
      * the tensor core, per MMA instruction of K_inst products on the running
        in-block sum s: every term truncated to 2^(e_max - 25) with 2^e_max <=
        max(|s|, max |term|) (raw product exponents never exceed the true ones),
        at most K_inst + 1 terms -> (K_inst + 1) * u/2 * max(|s|, max|term|); the
        RZ of the result < 2 u |s_after|; plus (K_inst + 1) * 2^-158 (J_min);
        D_corr's instructions P2, P3 the same, scaled by 2^-11 (FP16) / 1 (TF32);
      * the "ideal" side's one RN per block sum: u |P1_b| + scale * u |corr_b|;
      * t = RN(P1 + scale * corr) on both sides: 2 u |t_b|;
      * C = RN(C + t) on both sides: 2 u |C_b| (running sums, not |A||B|).
    The partial sums are taken from the exact products (float64), so the
    bound scales with the cancellation-aware |s| and |C_b|, not with |A||B|."""
    kinst = 16 if mode in (0, "fp16") else 8
    sc = 2.0 ** -11 if mode in (0, "fp16") else 1.0
    a = np.ascontiguousarray(a, dtype=np.float32)
    b = np.ascontiguousarray(b, dtype=np.float32)
    E, k = a.shape
    out = np.zeros(E)
    if k == 0 or E == 0:
        return out
    nb = -(-k // kb)
    ni = kb // kinst
    kp = nb * kb
    chunk = max(1, (1 << 21) // kp)
    for e0 in range(0, E, chunk):
        ha, la = (np.asarray(v, dtype=np.float64) for v in oracle.split_values(mode, a[e0:e0 + chunk]))
        hb, lb = (np.asarray(v, dtype=np.float64) for v in oracle.split_values(mode, b[e0:e0 + chunk]))
        e = ha.shape[0]

        def blocks(x):
            y = np.zeros((e, kp))
            y[:, :k] = x
            return y.reshape(e, nb, ni, kinst)

        # instructions that exist (the padding past k issues none)
        live = (np.arange(nb)[:, None] * kb + np.arange(ni)[None, :] * kinst) < k

        def instr_err(t, rep=1):    # t: (e, nb, rep * n_instr, K) exact terms in instruction order
            sa = np.cumsum(t.sum(-1), axis=-1)
            sb = np.concatenate([np.zeros(sa.shape[:-1] + (1,)), sa[..., :-1]], axis=-1)
            mx = np.maximum(np.abs(sb), np.abs(t).sum(-1))    # sum |terms| >= max |term|
            err = (kinst + 1) * (U / 2) * mx + 2 * U * np.abs(sa) + (kinst + 1) * JMIN_GRID
            return (err * np.repeat(live, rep, axis=1)).sum(-1), sa[..., -1]

        fin = np.all(np.isfinite(ha) & np.isfinite(hb) & np.isfinite(la) & np.isfinite(lb), axis=1)
        with np.errstate(invalid="ignore", over="ignore"):
            e1, p1 = instr_err(blocks(ha * hb))
            tot = e1 + U * np.abs(p1)
            t = p1
            if corr:
                q = np.stack([blocks(la * hb), blocks(ha * lb)], axis=3).reshape(e, nb, 2 * ni, kinst)
                ec, pc = instr_err(q, 2)
                tot = tot + sc * (ec + U * np.abs(pc))
                t = p1 + sc * pc
            cb = np.cumsum(t, axis=1)
            tot = tot + 2 * U * np.abs(t) + 2 * U * np.abs(cb)
            r = 1.02 * tot.sum(1)
        out[e0:e0 + e] = np.where(fin, r, np.inf)
    return out


def matrix_bound(mode, ar, bc, kb, corr=True):
    """entry_bound for every output of one problem at once: ar = rows of A (m, k),
    bc = columns of B (n, k); returns (n, m).  Same terms, with the
    per-instruction partial sums formed by (n x K_inst) @ (K_inst x m) products."""
    kinst = 16 if mode in (0, "fp16") else 8
    sc = 2.0 ** -11 if mode in (0, "fp16") else 1.0
    m, k = ar.shape
    n = bc.shape[0]
    if k == 0:
        return np.zeros((n, m))
    ha, la = (np.asarray(v, dtype=np.float64) for v in oracle.split_values(mode, ar))
    hb, lb = (np.asarray(v, dtype=np.float64) for v in oracle.split_values(mode, bc))
    fin = np.isfinite(hb).all(1)[:, None] & np.isfinite(lb).all(1)[:, None] & \
        np.isfinite(ha).all(1)[None, :] & np.isfinite(la).all(1)[None, :]
    ha, la, hb, lb = (np.nan_to_num(x, nan=0.0, posinf=0.0, neginf=0.0) for x in (ha, la, hb, lb))
    aha, ala, ahb, alb = np.abs(ha), np.abs(la), np.abs(hb), np.abs(lb)
    tot = np.zeros((n, m))
    cb = np.zeros((n, m))

    def step(acc, err, x, y, ax, ay):        # one instruction on the running sum acc
        t = x @ y.T
        mx = np.maximum(np.abs(acc), ax @ ay.T)
        acc = acc + t
        err += (kinst + 1) * (U / 2) * mx + 2 * U * np.abs(acc) + (kinst + 1) * JMIN_GRID
        return acc

    for p0 in range(0, k, kb):
        s = np.zeros((n, m))
        es = np.zeros((n, m))
        c = np.zeros((n, m))
        ec = np.zeros((n, m))
        for q0 in range(p0, min(p0 + kb, k), kinst):
            I = slice(q0, min(q0 + kinst, p0 + kb, k))
            s = step(s, es, hb[:, I], ha[:, I], ahb[:, I], aha[:, I])
            if corr:
                c = step(c, ec, hb[:, I], la[:, I], ahb[:, I], ala[:, I])     # P2 = lo_a hi_b
                c = step(c, ec, lb[:, I], ha[:, I], alb[:, I], aha[:, I])     # P3 = hi_a lo_b
        t = s + sc * c
        tot += es + U * np.abs(s) + sc * (ec + U * np.abs(c)) + 2 * U * np.abs(t)
        cb += t
        tot += 2 * U * np.abs(cb)
    return np.where(fin, 1.02 * tot, np.inf)


def tolerance(mode, A, B, m, n, k, kblock=0, corr=True, alpha=1.0, beta=0.0, C=None, range_safe=False):
    """Element-wise bar |C_gpu - C_oracle("ideal")| <= tol on
    column-major batched operands; returns (batch, n, m).  range_safe: the
    bound of the scaled problem (R#22) times 2^(e_i + f_j), plus the final
    unscaling's rounding."""
    kb = kblock or oracle.default_kb(k)
    A = np.asarray(A, dtype=np.float32)
    B = np.asarray(B, dtype=np.float32)
    if A.ndim == 2:
        A = A[None]
    if B.ndim == 2:
        B = B[None]
    batch = max(A.shape[0], B.shape[0])
    out = np.empty((batch, n, m))
    for bi in range(batch):
        Ab = A[bi if A.shape[0] > 1 else 0]
        Bb = B[bi if B.shape[0] > 1 else 0]
        ar = np.ascontiguousarray(Ab[:k, :m].T)          # rows of A (m, k)
        bc = np.ascontiguousarray(Bb[:n, :k])            # columns of B (n, k)
        if range_safe:
            ex, fx = oracle.range_exponents(Ab, Bb, m, n, k)
            ar = np.ldexp(ar, -ex[:, None].astype(np.int32)).astype(np.float32)
            bc = np.ldexp(bc, -fx[:, None].astype(np.int32)).astype(np.float32)
        out[bi] = matrix_bound(mode, ar, bc, kb, corr)
        if range_safe:
            out[bi] *= np.ldexp(1.0, (fx[:, None] + ex[None, :]).astype(np.int64))
        if range_safe or alpha != 1.0 or beta != 0.0:
            R = oracle.gemm_f64(Ab[None], Bb[None], m, n, k)[0]
            c0 = 0.0 if C is None or beta == 0.0 else \
                np.asarray(C, dtype=np.float64).reshape(batch, n, -1)[bi, :, :m]
            out[bi] = abs(alpha) * out[bi] * 1.01 + 2 * U * (abs(alpha) * np.abs(R) + np.abs(beta * c0)) + 1e-45
    return out


def tolerance_entries(mode, A, B, k, bidx, ii, jj, kblock=0, corr=True):
    """the same bar for sampled outputs C_{bidx}(ii, jj) (alpha = 1, beta = 0)"""
    kb = kblock or oracle.default_kb(k)
    A = np.asarray(A, dtype=np.float32)
    B = np.asarray(B, dtype=np.float32)
    sa = A.shape[0] > 1
    sb = B.shape[0] > 1
    a = np.stack([A[b if sa else 0, :k, i] for b, i in zip(bidx, ii)])
    bv = np.stack([B[b if sb else 0, j, :k] for b, j in zip(bidx, jj)])
    return entry_bound(mode, a, bv, kb, corr)


def emu_gpu_range(mode, A, B, m, n, k, alpha=1.0, beta=0.0, C=None, kblock=0, flags=0, range_flag=None):
    """the range-safe entry (R#22) on column-major numpy operands; returns (batch, n, m)"""
    import torch
    import paper_2308_15152_b200 as emu
    A = np.ascontiguousarray(A, dtype=np.float32)
    B = np.ascontiguousarray(B, dtype=np.float32)
    if A.ndim == 2:
        A = A[None]
    if B.ndim == 2:
        B = B[None]
    batch = max(A.shape[0], B.shape[0])
    lda, ldb = A.shape[2], B.shape[2]
    sA = 0 if (A.shape[0] == 1 and batch > 1) else A.shape[1] * lda
    sB = 0 if (B.shape[0] == 1 and batch > 1) else B.shape[1] * ldb
    dA = torch.from_numpy(A).cuda()
    dB = torch.from_numpy(B).cuda()
    if C is None:
        dC = torch.full((batch, n, m), float("nan"), device="cuda")
    else:
        dC = torch.from_numpy(np.ascontiguousarray(C, dtype=np.float32).reshape(batch, n, m)).cuda()
    nbytes = emu.emu_range_workspace_size(m, n, batch)
    ws = torch.empty(max(nbytes // 4, 4), dtype=torch.int32, device="cuda")
    emu.emu_sgemm_batched_range(m, n, k, alpha, dA, lda, sA, dB, ldb, sB, beta, dC, m, n * m, batch,
                                mode, ws, nbytes, None, range_flag, kblock, flags)
    torch.cuda.synchronize()
    return dC.cpu().numpy()
