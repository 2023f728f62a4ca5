"""The tile schedule does not change any output bit (dynamic tile order):
the long-k streaming path with the cluster-launch-control order (default) and with the
static order (EMU_TS_CLC=0, read once per process, hence the subprocesses) on a problem
with more tiles than resident clusters, so tiles really are taken over by try_cancel;
both bit-exact with the oracle's tensor-core model on sampled outputs."""
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle
import workloads
from gpu_util import assert_bits_equal

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# 9 m-pairs x 11 n-tiles = 99 tiles (> 74 clusters), ragged m / n / k, k >= 2048 (long-k rings)
SHAPES = [(1, 2048 + 64, 1280 + 40, 2048 + 96), (3, 1024, 1024, 2048),
          (1, 512, 4736, 2048),         # 74 tiles: every cluster resident, nothing to take over
          (1, 768, 3200, 2048 + 32)]    # 75 tiles: one more than the resident clusters

_RUN = r"""
import sys, numpy as np
sys.path.insert(0, {root!r}); sys.path.insert(0, {tests!r})
import workloads
from gpu_util import emu_gpu
import paper_2308_15152_b200 as emu
A, B = workloads.make_operands({batch}, {m}, {n}, {k}, seed={seed})
C = emu_gpu({mode!r}, A, B, {m}, {n}, {k})
np.save({out!r}, C)
print(emu.emu_last_kernel_name())
"""


def _run(tmp_path, tag, env_clc, mode, batch, m, n, k, seed):
    out = str(tmp_path / f"C_{tag}.npy")
    code = _RUN.format(root=ROOT, tests=os.path.join(ROOT, "tests"), batch=batch, m=m, n=n, k=k, seed=seed,
                       mode=mode, out=out)
    env = dict(os.environ)
    env.pop("EMU_TS_CLC", None)
    if env_clc is not None:
        env["EMU_TS_CLC"] = env_clc
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return np.load(out), r.stdout.strip().splitlines()[-1]


@pytest.mark.parametrize("mode", ["fp16", "tf32"])
@pytest.mark.parametrize("shape", SHAPES, ids=["ragged-99tiles", "batch3-96tiles", "74tiles", "75tiles"])
def test_dynamic_tile_order_bit_identical(tmp_path, mode, shape):
    batch, m, n, k = shape
    seed = 11
    c_dyn, name_dyn = _run(tmp_path, "dyn", None, mode, batch, m, n, k, seed)
    c_sta, name_sta = _run(tmp_path, "static", "0", mode, batch, m, n, k, seed)
    assert "long-k rings" in name_dyn and "long-k rings" in name_sta, (name_dyn, name_sta)
    assert "dynamic tile order" in name_dyn and "dynamic tile order" not in name_sta, (name_dyn, name_sta)
    assert_bits_equal(c_dyn, c_sta)
    A, B = workloads.make_operands(batch, m, n, k, seed=seed)
    g = workloads.rng(seed + 1)
    b, i, j = g.integers(0, batch, 64), g.integers(0, m, 64), g.integers(0, n, 64)
    # the last row / column of the ragged edges too
    b, i, j = np.append(b, [batch - 1, 0]), np.append(i, [m - 1, m - 1]), np.append(j, [n - 1, 0])
    assert_bits_equal(c_dyn[b, j, i], oracle.emu_gemm_entries(mode, A, B, m, n, k, b, i, j, tc="sm100"))


def test_dynamic_tile_order_two_streams():
    """two long-k GEMMs launched on two streams at once: each grid's clusters take over
    only their own grid's tiles (cluster launch control is per grid); both results equal
    the same GEMMs run one after the other"""
    import torch
    import paper_2308_15152_b200 as emu
    m, n, k, batch = 1024, 1280, 2048, 2
    ops = [workloads.make_operands(batch, m, n, k, seed=s) for s in (21, 22)]
    dev = [(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()) for A, B in ops]

    def run(dA, dB, stream):
        dC = torch.full((batch, n, m), float("nan"), device="cuda")
        st = emu.emu_sgemm_batched(m, n, k, 1.0, dA, m, k * m, dB, k, n * k, 0.0, dC, m, n * m, batch, "fp16",
                                   stream)
        assert "long-k rings" in emu.emu_last_kernel_name()
        return dC, st

    ref = []
    for dA, dB in dev:
        dC, _ = run(dA, dB, torch.cuda.current_stream())
        ref.append(dC)
    torch.cuda.synchronize()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize()
    with torch.cuda.stream(s1):
        c1, _ = run(*dev[0], s1)
    with torch.cuda.stream(s2):
        c2, _ = run(*dev[1], s2)
    torch.cuda.synchronize()
    assert_bits_equal(c1.cpu().numpy(), ref[0].cpu().numpy())
    assert_bits_equal(c2.cpu().numpy(), ref[1].cpu().numpy())
