"""The tensor core's accumulator, measured by the STANDALONE tcgen05 probe
(probe/tc_probe.cu: its own PTX, no code shared with libemusgemm) and compared
bit for bit with the oracle's instruction-level model (oracle.tc_chain,
oracle.c tc_instr; R#9).  The paper fixes only "RZ" (§4.4);
SPEC.md S:213 gives the vector that tells RZ from RN.

Every (kind, cta_group, A source) variant of tcgen05.mma the product uses (and
the ones it does not) runs every operand family of probe/families.py.  The
samples are written to gpurun_out/tcprobe/ for tools/tc_fit.py, which fits the
model to them alone."""
import os

import numpy as np
import pytest

import oracle
import probe
from probe import families

pytestmark = pytest.mark.gpu

VARIANTS = [(kind, pair, atm) for kind in ("fp16", "tf32") for pair in (0, 1) for atm in (0, 1)]
GRID = 8
SEED = 2308


def _vid(v):
    return f"{v[0]}-{'cta2' if v[1] else 'cta1'}-{'tmemA' if v[2] else 'smemA'}"


@pytest.fixture(scope="module", autouse=True)
def _built():
    probe.build()


@pytest.mark.parametrize("variant", VARIANTS, ids=_vid)
def test_probe_exact_integers(variant):
    """the probe itself: small-integer operands have exact sums, so D must be
    the float64 product whatever the accumulator does (checks the probe's
    layouts and descriptors before any model is compared)"""
    kind, pair, atm = variant
    rng = np.random.default_rng(7)
    K = families.KINST[kind]
    M = 256 if pair else 128
    n = 3
    A = rng.integers(-8, 9, size=(2, n, M, K)).astype(np.float32)
    B = rng.integers(-8, 9, size=(2, n, 64, K)).astype(np.float32)
    D0 = rng.integers(-100, 101, size=(2, M, 64)).astype(np.float32)
    D = probe.run(kind, pair, atm, A, B, D0)
    want = np.einsum("gimk,gink->gmn", A.astype(np.float64), B.astype(np.float64)) + D0
    assert np.array_equal(D.astype(np.float64), want)


def _save(variant, family, A, B, D0, D):
    """a subset of the samples (first problem; rows from both CTAs of a pair,
    columns from both halves of N) for tools/tc_fit.py and the CPU replay"""
    kind, pair, atm = variant
    rows = np.r_[0:32, 128:160] if pair else np.r_[0:64]
    cols = np.r_[0:16, 32:48]
    if family in ("subnorm", "subtie"):    # results in binary32's subnormal range: keep them all
        rows, cols = np.r_[0:A.shape[2]], np.r_[0:B.shape[2]]
    d = os.path.join("gpurun_out", "tcprobe")
    os.makedirs(d, exist_ok=True)
    np.savez_compressed(
        os.path.join(d, f"{_vid(variant)}-{family}.npz"),
        A=probe.operand_bits(kind, A[0][:, rows]), B=probe.operand_bits(kind, B[0][:, cols]),
        D0=(np.zeros((len(rows), len(cols)), np.float32) if D0 is None else D0[0][np.ix_(rows, cols)]),
        D=D[0][np.ix_(rows, cols)], meta=np.array([0 if kind == "fp16" else 1, pair, atm]))


@pytest.mark.parametrize("family", families.FAMILIES)
@pytest.mark.parametrize("variant", VARIANTS, ids=_vid)
def test_probe_vs_oracle_model(variant, family):
    kind, pair, atm = variant
    A, B, D0 = families.make(family, kind, pair, GRID, SEED)
    D = probe.run(kind, pair, atm, A, B, D0)
    _save(variant, family, A, B, D0, D)
    nbad = 0
    first = None
    for g in range(GRID):
        want = oracle.tc_chain(kind, A[g], B[g], None if D0 is None else D0[g], tc="sm100")
        bad = D[g].view(np.uint32) != want.view(np.uint32)
        bad &= ~((D[g] == 0) & (want == 0))      # +0 / -0 compare equal by value
        if bad.any() and first is None:
            r, j = np.argwhere(bad)[0]
            first = (g, int(r), int(j), float(D[g][r, j]).hex(), float(want[r, j]).hex())
        nbad += int(bad.sum())
    assert nbad == 0, f"{nbad} of {D.size} probe outputs differ from oracle tc_instr; first {first}"


@pytest.mark.parametrize("kind", ["fp16", "tf32"])
def test_s213_reading_is_rz(kind):
    """1 + 3*2^-24 in one instruction -> 1 + 2^-23 (RZ), not 1 + 2^-22 (RN)"""
    K = families.KINST[kind]
    A = np.zeros((1, 1, 128, K), np.float32)
    B = np.zeros((1, 1, 16, K), np.float32)
    A[..., 0], A[..., 1] = 1.0, 3 * 2.0 ** -12
    B[..., 0], B[..., 1] = 1.0, 2.0 ** -12
    D = probe.run(kind, 0, 0, A, B)
    assert np.all(D == np.float32(1 + 2.0 ** -23)), np.unique(D)
    D = probe.run(kind, 0, 0, -A, B)
    assert np.all(D == np.float32(-1 - 2.0 ** -23)), np.unique(D)
