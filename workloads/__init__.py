"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and
bench.py.  Holds NONE of the method's arithmetic (no split, no product, no
rounding model): only random numbers and shapes.  Both sides import this
module; neither side imports the other.

Storage convention (BLAS column-major, paper P:478 / DESIGN.md R#17): an m x k
matrix X with leading dimension ld is stored so that X(i, p) = buf[i + p*ld].
As numpy we hold it as an array of shape (k, ld) (C-contiguous), i.e. the
row index of the numpy array is the *column* of the matrix; batched operands
are (batch, k, ld).  `math_view` returns the m x k matrix view.

Recipes: every value is drawn from numpy's counter-based
Philox generator keyed by the seed, so every process/rank regenerates the
same data.
"""
from __future__ import annotations

import dataclasses
import numpy as np

__all__ = [
    "rng", "uniform", "log_uniform", "small_int", "colmajor", "math_view",
    "Config", "CONFIGS", "make_operands", "unit_vectors", "rotations",
]


def rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.Philox(key=int(seed)))


def uniform(shape, seed: int, lo: float = -1.0, hi: float = 1.0) -> np.ndarray:
    """uniform[lo, hi) float32 (north_star: inputs uniform in [-1, 1])."""
    g = rng(seed)
    x = g.random(size=shape, dtype=np.float32)
    return (x * np.float32(hi - lo) + np.float32(lo)).astype(np.float32)


def log_uniform(shape, seed: int, emin: float, emax: float) -> np.ndarray:
    """+-2^U(emin, emax) with a random sign (config c4: magnitudes spanning
    2^-30 .. 2^30).  Computed in float64, rounded once to float32."""
    g = rng(seed)
    e = g.uniform(emin, emax, size=shape)
    s = np.where(g.random(size=shape) < 0.5, -1.0, 1.0)
    return (s * np.exp2(e)).astype(np.float32)


def small_int(shape, seed: int, lo: int = -16, hi: int = 16) -> np.ndarray:
    """integers in [lo, hi] as float32 (exact-product pins)."""
    g = rng(seed)
    return g.integers(lo, hi + 1, size=shape).astype(np.float32)


def colmajor(math: np.ndarray, ld: int | None = None) -> np.ndarray:
    """m x k math matrix (or batch x m x k) -> column-major storage (.., k, ld)."""
    m = math.shape[-2]
    ld = m if ld is None else ld
    out = np.zeros(math.shape[:-2] + (math.shape[-1], ld), dtype=np.float32)
    out[..., :, :m] = np.swapaxes(math, -1, -2)
    return out


def math_view(store: np.ndarray, rows: int) -> np.ndarray:
    """column-major storage (.., cols, ld) -> (.., rows, cols) math view."""
    return np.swapaxes(store[..., :, :rows], -1, -2)


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    batch: int
    m: int
    n: int
    k: int
    dist: str          # "uniform" | "logu30" | "logu15"
    seed: int
    note: str


# BASELINE.json "configs" (c1..c5); shapes fixed there, seeds/distributions
# fixed here.
CONFIGS = {
    "c1": Config("c1", 16, 64, 64, 64, "uniform", 42,
                 "batched 16 x 64^3, uniform[-1,1] (oracle in seconds)"),
    "c2": Config("c2", 1024, 256, 256, 256, "uniform", 1,
                 "batched 1024 x 256^3, uniform[-1,1]"),
    "c3": Config("c3", 1, 16384, 16384, 16384, "uniform", 7,
                 "single 16384^3, uniform[-1,1]"),
    "c4": Config("c4", 1, 1024, 1024, 4096, "logu30", 11,
                 "k=4096, magnitudes 2^-30..2^30"),
    "c5": Config("c5", 8192, 256, 256, 256, "uniform", 5,
                 "8192 x 256^3 batch-sharded over ranks"),
}


def _draw(shape, seed, dist):
    if dist == "uniform":
        return uniform(shape, seed)
    if dist == "logu30":
        return log_uniform(shape, seed, -30.0, 30.0)
    if dist == "logu15":
        return log_uniform(shape, seed, -30.0, 15.0)
    if dist == "int16":
        return small_int(shape, seed)
    raise ValueError(dist)


def make_operands(batch: int, m: int, n: int, k: int, seed: int,
                  dist: str = "uniform", item0: int = 0, lda=None, ldb=None):
    """Column-major batched operands A (batch, k, lda), B (batch, n, ldb).

    Item b of the returned batch is global item (item0 + b); every item has
    its own seed stream (seed, item, operand), so a rank that generates items
    [r*B/G, (r+1)*B/G) sees exactly the data of the 1-GPU run.
    """
    lda = m if lda is None else lda
    ldb = k if ldb is None else ldb
    A = np.zeros((batch, k, lda), dtype=np.float32)
    B = np.zeros((batch, n, ldb), dtype=np.float32)
    for b in range(batch):
        g = item0 + b
        A[b, :, :m] = _draw((k, m), (seed * 1000003 + g) * 2 + 0, dist)
        B[b, :, :k] = _draw((n, k), (seed * 1000003 + g) * 2 + 1, dist)
    return A, B


def unit_vectors(batch: int, m: int, seed: int) -> np.ndarray:
    """(batch, m) float32 Householder vectors: uniform[-1,1] directions scaled
    to unit 2-norm in float64, rounded once to float32 (so ||v|| = 1 + O(u))."""
    x = uniform((batch, m), seed).astype(np.float64)
    x /= np.linalg.norm(x, axis=1, keepdims=True)
    return x.astype(np.float32)


def rotations(batch: int, seed: int) -> np.ndarray:
    """(batch, 2) float32 (c, s) = (cos t, sin t), t uniform in [0, 2 pi)."""
    t = rng(seed).uniform(0.0, 2.0 * np.pi, size=batch)
    return np.stack([np.cos(t), np.sin(t)], axis=1).astype(np.float32)
