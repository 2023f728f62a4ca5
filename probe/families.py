"""Seeded operand families for the tcgen05 accumulator probe (inputs only: no
arithmetic of the method here).  Every operand is an exact binary16 / TF32
value; each family targets one part of the accumulator's behaviour:

  s213      the SPEC.md S:213 vector -- products 1 and 3*2^-24 in one
            instruction (RZ -> 1 + 2^-23, RN -> 1 + 2^-22), random sign,
            scale and position, plus extra small terms
  alignS    11-bit significands, exponents uniform in [-S, S], random signs,
            5 % zeros (the alignment / guard-bit width)
  positive  as align12 with all products positive (truncation direction)
  cancel    x*y - x*y exactly (and x*y - x*y' with y' one operand ulp below y) plus small terms:
            does the alignment use the cancelled terms' exponent?
  subnorm   binary16 subnormal operands mixed with normal ones (fp16), or
            TF32 values whose products land in binary32's subnormal range
  subtie    TF32: sums in binary32's subnormal range built from 4-bit
            significands, so that many land exactly halfway between two
            subnormals (ties) or just beside halfway (an extra tiny term);
            binary16: as subnorm
  acc       an accumulator input D0 with a full 24-bit significand and
            magnitude 2^U(-30, 30) relative to the products
  chain     4-8 chained instructions (accumulation in tensor memory between
            instructions), with and without D0
Each returns (A (grid, n, M, K), B (grid, n, N, K), D0 (grid, M, N) | None).
"""
from __future__ import annotations

import numpy as np

FAMILIES = ["s213", "align1", "align3", "align6", "align12", "align24", "positive", "cancel",
            "subnorm", "subtie", "acc", "chain", "chain_acc"]
KINST = {"fp16": 16, "tf32": 8}


def _sig11(rng, shape):
    return rng.integers(1024, 2048, size=shape).astype(np.float64)


def _vals(rng, shape, emin, emax, kind, pzero=0.05, signed=True):
    """random exact values: 11-bit significand, exponent uniform in [emin, emax]"""
    x = np.ldexp(_sig11(rng, shape), rng.integers(emin, emax + 1, size=shape) - 10)
    if signed:
        x *= rng.choice([-1.0, 1.0], size=shape)
    x[rng.random(shape) < pzero] = 0.0
    return _exact(x, kind)


def _exact(x, kind):
    x = np.asarray(x, dtype=np.float64)
    if kind == "fp16":
        assert np.all(np.abs(x) <= 65504)
        y = x.astype(np.float16).astype(np.float64)
    else:
        y = x.astype(np.float32)
        b = y.view(np.uint32)
        assert not np.any(b & 0x1FFF)
        y = y.astype(np.float64)
    assert np.array_equal(y, x), "generator produced an inexact operand"
    return x.astype(np.float32)


def _one_ulp_less(y, kind):
    """the next operand value toward zero (y != 0)"""
    if kind == "fp16":
        return (y.astype(np.float16).view(np.uint16) - 1).view(np.float16).astype(np.float32)
    return (y.astype(np.float32).view(np.uint32) - 0x2000).view(np.float32)


def make(family, kind, pair, grid, seed, N=64):
    rng = np.random.default_rng([seed, FAMILIES.index(family), 0 if kind == "fp16" else 1, int(pair)])
    K = KINST[kind]
    M = 256 if pair else 128
    fp16 = kind == "fp16"
    n = 1
    D0 = None
    if family == "s213":
        A = np.zeros((grid, n, M, K))
        B = np.zeros((grid, n, N, K))
        sr = rng.integers(-6, 7, size=(grid, M)) if fp16 else rng.integers(-40, 41, size=(grid, M))
        sc = rng.integers(-6, 7, size=(grid, N)) if fp16 else rng.integers(-40, 41, size=(grid, N))
        for g in range(grid):
            perm = rng.permutation(K)
            # products: 1, 3*2^-24 and (K-2) terms 2^-24 * {0..3} * small
            a = np.zeros(K)
            b = np.zeros(K)
            a[perm[0]], b[perm[0]] = 1.0, 1.0
            a[perm[1]], b[perm[1]] = 3 * 2.0 ** -12, 2.0 ** -12
            extra = rng.integers(0, 4, size=K - 2)
            a[perm[2:]] = extra * 2.0 ** -13
            b[perm[2:]] = 2.0 ** -13
            sgn_r = rng.choice([-1.0, 1.0], size=M)
            sgn_c = rng.choice([-1.0, 1.0], size=N)
            A[g, 0] = (sgn_r * np.ldexp(1.0, sr[g]))[:, None] * a[None, :]
            B[g, 0] = (sgn_c * np.ldexp(1.0, sc[g]))[:, None] * b[None, :]
        return _exact(A, kind), _exact(B, kind), None
    if family.startswith("align") or family == "positive":
        S = 12 if family == "positive" else int(family[5:])
        lo, hi = (-min(S, 14), min(S, 14)) if fp16 else (-S, S)   # binary16: normal range
        signed = family != "positive"
        A = _vals(rng, (grid, n, M, K), lo, hi, kind, signed=signed)
        B = _vals(rng, (grid, n, N, K), lo, hi, kind, signed=signed)
        return A, B, None
    if family == "cancel":
        A = _vals(rng, (grid, n, M, K), -12, -2, kind)
        B = _vals(rng, (grid, n, N, K), -12, -2, kind)
        for g in range(grid):
            p, q = rng.choice(K, size=2, replace=False)
            x = _vals(rng, (M,), 0, 6, kind, pzero=0.0)
            y = _vals(rng, (N,), 0, 6, kind, pzero=0.0)
            A[g, 0, :, p] = x
            A[g, 0, :, q] = x
            B[g, 0, :, p] = y
            near = rng.random(N) < 0.5
            B[g, 0, :, q] = np.where(near, -_one_ulp_less(y, kind), -y)
        return A, B, None
    if family == "subnorm":
        if fp16:
            # binary16 subnormals m * 2^-24 (m < 1024) and small normals, some large terms
            sub = rng.integers(1, 1024, size=(grid, n, M, K)) * 2.0 ** -24
            A = np.where(rng.random((grid, n, M, K)) < 0.6, sub * rng.choice([-1.0, 1.0], size=sub.shape),
                         _vals(rng, (grid, n, M, K), -14, -8, kind))
            subb = rng.integers(1, 1024, size=(grid, n, N, K)) * 2.0 ** -24
            B = np.where(rng.random((grid, n, N, K)) < 0.3, subb,
                         _vals(rng, (grid, n, N, K), -14, 4, kind))
            return _exact(A, kind), _exact(B, kind), None
        # TF32: products in binary32's subnormal range (2^-149 .. 2^-126), and TF32 subnormal operands
        A = _vals(rng, (grid, n, M, K), -75, -64, kind)
        B = _vals(rng, (grid, n, N, K), -75, -64, kind)
        tiny = rng.random((grid, n, M, K)) < 0.2
        sub = rng.integers(1, 1024, size=(grid, n, M, K)) * 2.0 ** -136    # TF32 subnormals (low 13 bits 0)
        A = np.where(tiny, sub, A)
        # a third of the columns mix in large terms; the rest keep every product tiny
        big = (rng.random((grid, n, N, K)) < 0.2) & (rng.random((grid, n, N, 1)) < 0.33)
        B = np.where(big, _vals(rng, (grid, n, N, K), 60, 70, kind), B)
        return _exact(A, kind), _exact(B, kind), None
    if family == "subtie":
        if fp16:
            return make("subnorm", kind, pair, grid, seed + 1, N)
        # a = +-(1 + i/8) 2^ea: products are multiples of 2^(ea+eb-6); ea + eb in [-144, -141]
        # puts them on a 2^-150 .. 2^-147 grid with magnitudes ~2^-144 .. 2^-139
        def few(shape, emin, emax):
            v = (1 + rng.integers(0, 8, size=shape) / 8.0) * np.ldexp(1.0, rng.integers(emin, emax + 1, size=shape))
            return v * rng.choice([-1.0, 1.0], size=shape)
        A = few((grid, n, M, K), -72, -70)
        B = few((grid, n, N, K), -72, -71)
        # slot K-1: a tiny extra term (2^-160 .. 2^-152) for half the rows x half the columns
        A[..., K - 1] = np.where(rng.random((grid, n, M)) < 0.5, few((grid, n, M), -82, -78), 0.0)
        B[..., K - 1] = np.where(rng.random((grid, n, N)) < 0.5, few((grid, n, N), -78, -74), 0.0)
        return _exact(A, kind), _exact(B, kind), None
    if family in ("acc", "chain", "chain_acc"):
        if family != "acc":
            n = int(rng.integers(4, 9))
        S = 3 if fp16 else 6
        A = _vals(rng, (grid, n, M, K), -S, S, kind)
        B = _vals(rng, (grid, n, N, K), -S, S, kind)
        if family in ("acc", "chain_acc"):
            sig = rng.integers(1 << 23, 1 << 24, size=(grid, M, N)).astype(np.float64)
            e = rng.integers(-30, 31, size=(grid, M, N))
            D0 = (np.ldexp(sig, e - 23) * rng.choice([-1.0, 1.0], size=sig.shape)).astype(np.float32)
            D0[rng.random(D0.shape) < 0.05] = 0.0
        return A, B, D0
    raise ValueError(family)
