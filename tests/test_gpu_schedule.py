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
SHAPES = [(1, 2048 + 64, 1280 + 40, 2048 + 96), (3, 1024, 1024, 2048)]

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
@pytest.mark.parametrize("shape", SHAPES, ids=["ragged-99tiles", "batch3-96tiles"])
def test_dynamic_tile_order_bit_identical(tmp_path, mode, shape):
    batch, m, n, k = shape
    seed = 11
    c_dyn, name_dyn = _run(tmp_path, "dyn", None, mode, batch, m, n, k, seed)
    c_sta, name_sta = _run(tmp_path, "static", "0", mode, batch, m, n, k, seed)
    assert "long-k rings" in name_dyn and "long-k rings" in name_sta, (name_dyn, name_sta)
    assert_bits_equal(c_dyn, c_sta)
    A, B = workloads.make_operands(batch, m, n, k, seed=seed)
    g = workloads.rng(seed + 1)
    b, i, j = g.integers(0, batch, 64), g.integers(0, m, 64), g.integers(0, n, 64)
    # the last row / column of the ragged edges too
    b, i, j = np.append(b, [batch - 1, 0]), np.append(i, [m - 1, m - 1]), np.append(j, [n - 1, 0])
    assert_bits_equal(c_dyn[b, j, i], oracle.emu_gemm_entries(mode, A, B, m, n, k, b, i, j, tc="sm100"))
