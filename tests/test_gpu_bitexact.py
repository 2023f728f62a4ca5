"""Bit-exact GPU parity against the oracle's measured tensor-core model.

The oracle's "sm100" model (oracle.c tc_instr, R#9) states how one
tcgen05.mma instruction adds its K_inst exact products to the FP32 accumulator
(alignment to the largest un-normalised exponent with 2 extra bits, truncation,
RZ -- the paper's "RZ" inside the Tensor Core).  With it, the whole
emulated GEMM (split, three products per K step, per-k-block outside combine,
epilogue) has one defined result per output, and the GPU must reproduce it bit
for bit.  These cases stress what the model has to get right: exponent spreads
(alignment), binary16 subnormal operands (the minimum exponent), long and
chunked k-blocks, ragged tails, every kernel the dispatch picks, transposed
operands, the range-safe mode and the BLAS epilogue.
"""
import numpy as np
import pytest

import oracle
import workloads
from gpu_util import assert_bits_equal, emu_gpu, emu_gpu_range, tolerance

pytestmark = pytest.mark.gpu
MODES = ["fp16", "tf32"]


def _logu(shape, lo, hi, seed):
    g = workloads.rng(seed)
    return (np.exp2(g.uniform(lo, hi, size=shape)) * g.choice([-1.0, 1.0], size=shape)).astype(np.float32)


def _check(mode, A, B, m, n, k, kblock=0, **kw):
    C = emu_gpu(mode, A, B, m, n, k, kblock=kblock, **kw)
    want = oracle.emu_gemm(mode, A, B, m, n, k, kb=kblock or oracle.default_kb(k), alpha=kw.get("alpha", 1.0),
                           beta=kw.get("beta", 0.0), C=kw.get("C"), corr=not (kw.get("flags", 0) & 1),
                           tc="sm100")
    assert_bits_equal(C[..., :m], want[..., :m])
    return C


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("m", [100, 300])        # single-CTA kernel / CTA-pair TS kernel
@pytest.mark.parametrize("spread", [(-1, 1), (-12, 12), (-20, 15)])
def test_exponent_spread(mode, m, spread):
    n, k = 136, 200
    A = _logu((1, k, m), *spread, seed=900 + m)
    B = _logu((1, n, k), *spread, seed=901 + m)
    _check(mode, A, B, m, n, k)


@pytest.mark.parametrize("mode", MODES)
def test_binary16_subnormal_operands(mode):
    """magnitudes 2^-24..2^-12: FP16 hi parts subnormal, lo parts mostly zero
    or subnormal -- the alignment exponent of a subnormal operand is e_min"""
    m, n, k = 256, 128, 128
    A = _logu((1, k, m), -24, -12, seed=910)
    B = _logu((1, n, k), -24, -8, seed=911)
    _check(mode, A, B, m, n, k)
    Am = _logu((1, k, m), -24, 2, seed=912)     # subnormal and normal terms mixed
    Bm = _logu((1, n, k), -24, 2, seed=913)
    _check(mode, Am, Bm, m, n, k)


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("kblock", [32, 64, 128, 256, 512])
def test_kblock_sweep(mode, kblock):
    """k-blocks of one to sixteen 32-k stages (longer than the operand ring on the
    TS kernel: issued in chunks, same per-accumulator order)"""
    m, n, k = 384, 256, 1000
    A, B = workloads.make_operands(1, m, n, k, seed=920 + kblock)
    _check(mode, A, B, m, n, k, kblock=kblock)


@pytest.mark.parametrize("mode", MODES)
def test_c2_items_astationary(mode):
    """c2's item shape (256^3) batched: the A-stationary TS path bench.py times"""
    A, B = workloads.make_operands(160, 256, 256, 256, seed=1)   # >= 148 row blocks: A-stationary
    C = emu_gpu(mode, A, B, 256, 256, 256)
    items = [0, 1, 77, 158, 159]
    want = oracle.emu_gemm(mode, A[items], B[items], 256, 256, 256, tc="sm100")
    assert_bits_equal(C[items], want)


@pytest.mark.parametrize("mode", MODES)
def test_ragged_epilogue_and_policy(mode):
    m, n, k, batch = 257, 129, 77, 3
    A, B = workloads.make_operands(batch, m, n, k, seed=930)
    C0 = workloads.uniform((batch, n, m), seed=931)
    _check(mode, A, B, m, n, k, alpha=-0.75, beta=1.25, C=C0)
    _check(mode, A, B, m, n, k, flags=1)       # correction off (P1 only)
    _check(mode, A, B, 1, 1, 1)
    _check(mode, A[:, :, :128], B, 128, n, k)  # m = 128 exactly: single-CTA kernel


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("trans", ["TN", "NT", "TT"])
def test_transposed(mode, trans):
    from test_gpu_trans import _gpu_t, _stored_t
    batch, m, n, k = 2, 200, 136, 300
    A, B = workloads.make_operands(batch, m, n, k, seed=940, lda=200, ldb=300)
    As = _stored_t(A) if trans[0] == "T" else A
    Bs = _stored_t(B) if trans[1] == "T" else B
    C = _gpu_t(mode, trans[0], trans[1], As, Bs, m, n, k)
    assert_bits_equal(C, oracle.emu_gemm(mode, A, B, m, n, k, tc="sm100"))


@pytest.mark.parametrize("mode", MODES)
def test_range_safe_mode(mode):
    """c4's magnitudes (2^-30..2^30) through the range-safe entry (R#22)"""
    m, n, k = 256, 192, 1024
    A = _logu((1, k, m), -30, 30, seed=950)
    B = _logu((1, n, k), -30, 30, seed=951)
    C = emu_gpu_range(mode, A, B, m, n, k)
    assert_bits_equal(C, oracle.emu_gemm_range(mode, A, B, m, n, k, tc="sm100"))


@pytest.mark.parametrize("mode", MODES)
def test_default_kblock_rule(mode):
    """kblock = 0 selects KB = 128 above k = 8192 (R#7): identical bits to an
    explicit 128, and to the oracle's own default"""
    m, n, k = 256, 128, 8224
    A, B = workloads.make_operands(1, m, n, k, seed=960)
    C = emu_gpu(mode, A, B, m, n, k)
    assert np.array_equal(C, emu_gpu(mode, A, B, m, n, k, kblock=128))
    assert_bits_equal(C, oracle.emu_gemm(mode, A, B, m, n, k, tc="sm100"))
    # model-free bars at this k: the element-wise bound against the ideal model
    # and north_star's accuracy gate (rel-Frobenius <= 2x plain FP32 SGEMM)
    d = np.abs(C.astype(np.float64) - oracle.emu_gemm(mode, A, B, m, n, k))
    assert np.all(d <= tolerance(mode, A, B, m, n, k))
    R = oracle.gemm_f64(A, B, m, n, k)
    assert oracle.rel_frobenius(C, R) <= 2 * oracle.rel_frobenius(oracle.sgemm_f32(A, B, m, n, k), R)


@pytest.mark.parametrize("mode", MODES)
def test_few_tiles_64_wide(mode):
    """fewer 256 x 128 tiles than clusters -> 64-wide tiles with double-buffered
    accumulators (c4's 1024^2 output); same bits as the oracle"""
    m, n, k = 384, 200, 500
    A, B = workloads.make_operands(1, m, n, k, seed=970)
    _check(mode, A, B, m, n, k)
    m, n, k = 1024, 1024, 4096        # c4's shape, sampled outputs
    A, B = workloads.make_operands(1, m, n, k, seed=971)
    C = emu_gpu(mode, A, B, m, n, k)
    g = workloads.rng(972)
    i, j = g.integers(0, m, 256), g.integers(0, n, 256)
    b = np.zeros(256, dtype=np.int64)
    assert_bits_equal(C[0, j, i], oracle.emu_gemm_entries(mode, A, B, m, n, k, b, i, j, tc="sm100"))


@pytest.mark.parametrize("mode", MODES)
def test_streaming_128_wide(mode):
    """enough tiles for every cluster but too few row blocks for A-stationary:
    the streaming-A split-commit 128-wide kernel"""
    batch, m, n, k = 40, 256, 256, 300
    A, B = workloads.make_operands(batch, m, n, k, seed=980)
    C = emu_gpu(mode, A, B, m, n, k)
    items = [0, 17, 39]
    assert_bits_equal(C[items], oracle.emu_gemm(mode, A[items], B[items], m, n, k, tc="sm100"))


@pytest.mark.parametrize("mode", MODES)
def test_c1_full(mode):
    """BASELINE.json configs[0]: 16 x 64^3 (single-CTA kernel), every output"""
    A, B = workloads.make_operands(16, 64, 64, 64, seed=42)
    _check(mode, A, B, 64, 64, 64)


@pytest.mark.parametrize("mode", MODES)
def test_c5_full_size_sampled(mode):
    """BASELINE.json configs[4]: 8192 x 256^3 in one launch (the 1-GPU share of the
    batch-sharded run); sampled outputs across the whole batch"""
    import torch
    import paper_2308_15152_b200 as emu
    batch, m, n, k = 8192, 256, 256, 256
    A, B = workloads.make_operands(batch, m, n, k, seed=5)
    dC = torch.empty((batch, n, m), device="cuda")
    emu.emu_sgemm_batched(m, n, k, 1.0, torch.from_numpy(A).cuda(), m, k * m, torch.from_numpy(B).cuda(), k,
                          n * k, 0.0, dC, m, n * m, batch, mode)
    torch.cuda.synchronize()
    g = workloads.rng(6)
    b, i, j = g.integers(0, batch, 512), g.integers(0, m, 512), g.integers(0, n, 512)
    b[0], i[0], j[0] = batch - 1, m - 1, n - 1
    got = dC[torch.from_numpy(b), torch.from_numpy(j), torch.from_numpy(i)].cpu().numpy()
    assert_bits_equal(got, oracle.emu_gemm_entries(mode, A, B, m, n, k, b, i, j, tc="sm100"))
