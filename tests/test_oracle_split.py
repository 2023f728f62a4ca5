"""Pins for the oracle's split (Eqs. corr-1..corr-4; reading R#6 for
TF32) against things other than itself: an independent binary16 conversion
(torch's CPU cast, exhaustively; numpy's cast on a sample), an independent
bit-pattern formula and float64 rint model for TF32, the SPEC worked vectors
(tests/golden/split_vectors.txt) and closed-form properties of the split."""
import concurrent.futures
import math
import os

import numpy as np
import pytest
import torch

import oracle
import workloads

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "split_vectors.txt")
CHUNK = 1 << 24


def _chunks():
    for c in range(0, 1 << 32, CHUNK):
        yield np.arange(c, c + CHUNK, dtype=np.uint64).astype(np.uint32)


def _exhaustive(check):
    """run check(u) over all 2^32 bit patterns in parallel chunks; sum counts"""
    nthr = max(1, min(8, os.cpu_count() or 1))
    saved = oracle.max_threads()
    oracle.set_threads(1)
    try:
        with concurrent.futures.ThreadPoolExecutor(nthr) as ex:
            starts = range(0, 1 << 32, CHUNK)
            return sum(ex.map(lambda c: check(np.arange(c, c + CHUNK, dtype=np.uint64)
                                              .astype(np.uint32)), starts))
    finally:
        oracle.set_threads(saved)


def test_f32_to_f16_exhaustive_vs_torch():
    """toFP16 == IEEE RNE binary16 (torch CPU cast) on all 2^32 inputs;
    NaNs compare by NaN-ness only."""
    torch.set_num_threads(1)

    def check(u):
        x = u.view(np.float32)
        ref = torch.from_numpy(x).to(torch.float16).view(torch.int16).numpy().view(np.uint16)
        hi, _ = oracle.split_fp16(x)
        nan = np.isnan(x)
        bad = int(np.count_nonzero((hi != ref) & ~nan))
        # NaN in -> NaN out
        hv = hi[nan]
        return bad + int(np.count_nonzero(((hv & 0x7c00) != 0x7c00) | ((hv & 0x3ff) == 0)))
    assert _exhaustive(check) == 0


def test_f32_to_f16_sample_vs_numpy():
    """a second independent implementation (numpy's float16 cast)."""
    g = workloads.rng(3)
    u = g.integers(0, 1 << 32, size=1 << 22, dtype=np.uint64).astype(np.uint32)
    # plus every pattern around the FP16 range edges and ties
    edges = np.array([0x33000000, 0x33000001, 0x387fe000, 0x387ff000, 0x38800000,
                      0x477fe000, 0x477fefff, 0x477ff000, 0x47800000, 0x3f801000,
                      0x3f803000, 0x3f800fff], dtype=np.uint32)
    u = np.concatenate([u, edges, edges | 0x80000000])
    x = u.view(np.float32)
    ref = x.astype(np.float16).view(np.uint16)
    hi, _ = oracle.split_fp16(x)
    ok = (hi == ref) | np.isnan(x)
    assert ok.all(), hex(int(u[~ok][0]))


def _tf32_bitformula(u):
    """RNE to 10 fraction bits on the binary32 bit pattern: add 0xfff plus the
    kept LSB, then clear the low 13 bits (carries propagate into the exponent
    and into Inf exactly as rounding does)."""
    r = u + np.uint32(0xfff) + ((u >> np.uint32(13)) & np.uint32(1))
    return r & np.uint32(0xffffe000)   # (finite inputs never wrap 32 bits)


def test_f32_to_tf32_exhaustive_vs_bitformula():
    def check(u):
        x = u.view(np.float32)
        hi, _ = oracle.split_tf32(x)
        fin = (u & np.uint32(0x7f800000)) != np.uint32(0x7f800000)
        ref = _tf32_bitformula(u)
        bad = int(np.count_nonzero((hi.view(np.uint32) != ref) & fin))
        # Inf -> Inf, NaN -> NaN
        return bad + int(np.count_nonzero(~fin & ~((hi.view(np.uint32) == u) | (np.isnan(hi) & np.isnan(x)))))
    assert _exhaustive(check) == 0


def test_f32_to_tf32_sample_vs_float64_rint():
    """TF32 == round-to-nearest-even to 11 significant bits with binary32's
    exponent range (quantum never below 2^-136), via float64 arithmetic."""
    g = workloads.rng(5)
    u = g.integers(0, 0x7f800000, size=1 << 20, dtype=np.uint64).astype(np.uint32)
    x = u.view(np.float32).astype(np.float64)
    ax = np.abs(x)
    with np.errstate(divide="ignore"):
        e = np.floor(np.log2(np.where(ax > 0, ax, 1.0)))
    q = np.exp2(np.maximum(e - 10, -136.0))
    ref = np.rint(x / q) * q
    ref = np.where(np.abs(ref) >= 2.0 ** 128, np.inf, ref)
    hi, _ = oracle.split_tf32(u.view(np.float32))
    assert np.array_equal(hi.astype(np.float64), ref)


def _golden():
    rows = []
    with open(GOLDEN) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            kind, inp, exp, cite = [s.strip() for s in line.split("|")]
            rows.append((kind, inp, exp, cite))
    return rows


@pytest.mark.parametrize("row", _golden(), ids=lambda r: f"{r[0]}:{r[1]}")
def test_golden_vectors(row):
    kind, inp, exp, cite = row
    ev = {"inf": math.inf}
    if kind == "f32_to_f16":
        hi, _ = oracle.split_values("fp16", np.array([eval(inp)], dtype=np.float32))
        assert hi[0] == np.float32(eval(exp)), cite
    elif kind == "f16_to_f32_bits":
        v = oracle.f16_bits_to_f32(np.array([eval(inp)]))[0]
        assert v == np.float32(eval(exp, ev)), cite
    elif kind == "split_fp16":
        hi, lo = oracle.split_values("fp16", np.array([eval(inp)], dtype=np.float32))
        eh, el = eval(exp)
        assert (hi[0], lo[0]) == (np.float32(eh), np.float32(el)), cite
    elif kind == "reconstruct_fp16":
        h, l = eval(inp)
        v = oracle.reconstruct("fp16", np.array([h], np.float32), np.array([l], np.float32))[0]
        assert v == np.float32(eval(exp)), cite
    elif kind == "tc_probe":
        pass  # used on the GPU (tests/test_gpu_probe.py)
    else:
        raise AssertionError(kind)


def _ulp32(x):
    return np.spacing(np.abs(x).astype(np.float32)).astype(np.float64)


def test_fp16_split_reconstruction_closed_forms():
    """On the FP16-normal range of the residual, [2^-13, 65504):
    (a) inputs with <= 22 significant bits reconstruct exactly;
    (b) every input reconstructs within 1 binary32 ulp (RNE hi => the residual
        fits 12 bits + sign, lo keeps 11 of them)."""
    g = workloads.rng(11)
    e = g.uniform(-13, math.log2(65504), size=1 << 20)
    x = (np.exp2(e) * np.where(g.random(1 << 20) < 0.5, -1, 1)).astype(np.float32)
    hi, lo = oracle.split_values("fp16", x)
    rec = oracle.reconstruct("fp16", hi, lo).astype(np.float64)
    err = np.abs(rec - x.astype(np.float64))
    assert np.all(err <= _ulp32(x))
    # (a) clear the two lowest significand bits -> <= 22 significant bits
    x22 = (x.view(np.uint32) & ~np.uint32(3)).view(np.float32)
    hi, lo = oracle.split_values("fp16", x22)
    assert np.array_equal(oracle.reconstruct("fp16", hi, lo), x22)


def test_fp16_split_structure():
    """hi is the RNE binary16 of x; lo*2^-11 is the RNE (binary16 grid, scaled)
    of the exact residual; x - hi is exact (R#2)."""
    x = workloads.uniform(1 << 18, seed=13)
    hi, lo = oracle.split_values("fp16", x)
    assert np.array_equal(hi, x.astype(np.float16).astype(np.float32))
    r = x.astype(np.float64) - hi.astype(np.float64)
    assert np.array_equal((r * 2048).astype(np.float16).astype(np.float64), lo.astype(np.float64))
    # |lo| <= 2^11 * half-ulp16(hi): the residual is at most half a binary16 ulp
    assert np.all(np.abs(r) <= np.spacing(np.abs(hi).astype(np.float16)).astype(np.float64) / 2 + 2.0 ** -25)


def test_fp16_split_special_values():
    """R#4/R#5: overflow and signed zero follow the IEEE evaluation of Eq.
    corr-1/corr-2: split(65519) = (65504, 15*2^11), split(65520) = (+Inf, -Inf),
    split(-0) = (-0, +0)."""
    x = np.array([65519.0, 65520.0, -0.0, np.inf, -np.inf], dtype=np.float32)
    hi, lo = oracle.split_fp16(x)
    assert list(hi[:3]) == [0x7bff, 0x7c00, 0x8000]
    assert list(lo[:3]) == [0x7780, 0xfc00, 0x0000]
    assert hi[3] == 0x7c00 and hi[4] == 0xfc00


def test_tf32_split_reconstruction():
    """TF32: hi + lo reconstructs x within 2^-21 relative (11 + 11 bits of a
    24-bit significand, both RNE)."""
    x = workloads.uniform(1 << 18, seed=17)
    hi, lo = oracle.split_tf32(x)
    assert np.all((hi.view(np.uint32) & 0x1fff) == 0)
    assert np.all((lo.view(np.uint32) & 0x1fff) == 0)
    rec = hi.astype(np.float64) + lo.astype(np.float64)
    nz = x != 0
    rel = np.abs(rec[nz] - x[nz]) / np.abs(x[nz].astype(np.float64))
    assert rel.max() <= 2.0 ** -21
