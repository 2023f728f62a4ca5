"""The C-ABI library loads, exports every symbol include/emu_sgemm.h declares,
and its host-side validation (which runs before any CUDA call) behaves as the
header documents.  No compute calls: no GPU here."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "emu_sgemm.h")


@pytest.fixture(scope="module")
def emu():
    import importlib.util
    spec = importlib.util.spec_from_file_location(
        "_emu_build", os.path.join(ROOT, "paper_2308_15152_b200", "build.py"))
    build = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(build)  # by path: the package import needs the .so first
    build.build()
    import paper_2308_15152_b200 as emu
    return emu


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(emu_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = _declared()
    for required in ["emu_sgemm", "emu_sgemm_batched", "emu_sgemm_batched_ex", "emu_split",
                     "emu_status_string", "emu_version", "emu_sgemm_batched_host"]:
        assert required in names


def test_library_exports_every_declared_symbol(emu):
    lib = ctypes.CDLL(emu.LIB_PATH)
    for name in _declared():
        assert hasattr(lib, name), name


def test_only_declared_symbols_are_exported(emu):
    out = os.popen(f"nm -D --defined-only {emu.LIB_PATH}").read()
    exported = {l.split()[-1] for l in out.splitlines() if " T " in l and l.split()[-1].startswith("emu_")}
    assert exported == set(_declared())


def test_library_is_sm100a_only(emu):
    out = os.popen(f"cuobjdump --list-elf {emu.LIB_PATH}").read()
    assert "sm_100a" in out
    assert all("sm_100a" in l for l in out.splitlines() if l.strip())


def test_status_strings_and_version(emu):
    for s in range(6):
        assert emu.emu_status_string(s).startswith("EMU_STATUS_")
    assert emu.emu_status_string(99) == "EMU_STATUS_UNKNOWN"
    assert emu.emu_version() >= 100


def _call(emu, **kw):
    a = dict(m=8, n=8, k=8, alpha=1.0, A=16, lda=8, strideA=0, B=16, ldb=8, strideB=0, beta=0.0,
             C=16, ldc=8, strideC=64, batch=1, mode=0)
    a.update(kw)
    return emu.lib.emu_sgemm_batched(a["m"], a["n"], a["k"], a["alpha"], a["A"], a["lda"], a["strideA"],
                                     a["B"], a["ldb"], a["strideB"], a["beta"], a["C"], a["ldc"],
                                     a["strideC"], a["batch"], a["mode"], None)


@pytest.mark.parametrize("kw", [dict(m=-1), dict(n=-1), dict(k=-1), dict(batch=-1), dict(mode=2),
                                dict(lda=7), dict(ldb=7), dict(ldc=7), dict(C=None),
                                dict(A=None), dict(B=None), dict(strideA=-4),
                                dict(batch=2, strideC=63)])
def test_invalid_arguments_rejected_before_launch(emu, kw):
    assert _call(emu, **kw) == 1   # EMU_STATUS_INVALID_VALUE


@pytest.mark.parametrize("kw", [dict(m=0), dict(n=0), dict(batch=0), dict(m=0, C=None)])
def test_quick_return_without_device(emu, kw):
    assert _call(emu, **kw) == 0
    assert emu.emu_last_launch_count() == 0
    assert isinstance(emu.emu_last_kernel_name(), str)


def test_ex_validation(emu):
    L = emu.lib
    args = [8, 8, 8, 1.0, 16, 8, 0, 16, 8, 0, 0.0, 16, 8, 0, 1, 0, None, None]
    assert L.emu_sgemm_batched_ex(*args, 48, 0) == 1      # kblock not a multiple of 32
    assert L.emu_sgemm_batched_ex(*args, -32, 0) == 1
    assert L.emu_sgemm_batched_ex(*args, 8192, 0) == 1
    assert L.emu_sgemm_batched_ex(*args, 0, 4) == 1       # unknown flag bit


def test_split_validation(emu):
    L = emu.lib
    assert L.emu_split(16, -1, 0, 16, 16, None) == 1
    assert L.emu_split(16, 4, 7, 16, 16, None) == 1
    assert L.emu_split(None, 4, 0, 16, 16, None) == 1
    assert L.emu_split(18, 4, 0, 16, 16, None) == 1       # misaligned
    assert L.emu_split(None, 0, 0, None, None, None) == 0


def test_range_entry_validation(emu):
    """range-safe entry (R#22): workspace size and the workspace checks run
    before any CUDA call."""
    L = emu.lib
    assert L.emu_range_workspace_size(256, 128, 10) == 4 * 10 * (256 + 128)
    assert L.emu_range_workspace_size(-1, 8, 1) == 0
    args = [8, 8, 8, 1.0, 16, 8, 0, 16, 8, 0, 0.0, 16, 8, 0, 1, 0, None]
    need = 4 * (8 + 8)
    assert L.emu_sgemm_batched_range(*args, None, need, None, 0, 0) == 1      # no workspace
    assert L.emu_sgemm_batched_range(*args, 4096, need - 4, None, 0, 0) == 1  # too small
    assert L.emu_sgemm_batched_range(*args, 4100, need, None, 0, 0) == 1     # not 16-byte aligned
    assert L.emu_sgemm_batched_range(*args, 4096, need, None, 48, 0) == 1    # kblock
    bad = list(args)
    bad[0] = -1
    assert L.emu_sgemm_batched_range(*bad, 4096, need, None, 0, 0) == 1
    empty = list(args)
    empty[14] = 0                                                             # batch = 0: quick return
    assert L.emu_sgemm_batched_range(*empty, 4096, 0, None, 0, 0) == 0


def test_transpose_entry_validation(emu):
    """emu_sgemm_batched_t: trans characters and the transposed leading-dimension
    rules are checked before any CUDA call (NEXT row 2)."""
    L = emu.lib
    base = dict(m=8, n=16, k=32, alpha=1.0, A=16, lda=8, sA=0, B=16, ldb=32, sB=0, beta=0.0, C=16, ldc=8,
                sC=0, batch=1, mode=0)

    def call(ta, tb, **kw):
        a = dict(base)
        a.update(kw)
        return L.emu_sgemm_batched_t(ta, tb, a["m"], a["n"], a["k"], a["alpha"], a["A"], a["lda"], a["sA"],
                                     a["B"], a["ldb"], a["sB"], a["beta"], a["C"], a["ldc"], a["sC"],
                                     a["batch"], a["mode"], None, None, 0, 0)
    assert call(b"X", b"N") == 1
    assert call(b"N", b"Q") == 1
    assert call(b"T", b"N", lda=8) == 1        # A stored k x m: lda >= k = 32
    assert call(b"N", b"T", ldb=8) == 1        # B stored n x k: ldb >= n = 16
    assert call(b"t", b"n", lda=32, batch=0) == 0   # valid, quick return
    assert call(b"C", b"c", lda=32, ldb=16, batch=0) == 0


def test_tcec_entries_validation(emu):
    """device-API users (NEXT rows 2 and 4): argument checks run before any CUDA call"""
    L = emu.lib
    g = [8, 8, 8, 1.0, 16, 8, 0, 16, 8, 0, 0.0, 16, 8, 0, 1, 0, None]
    assert L.emu_tcec_gemm_batched(*g, 0, 8) == 1            # unknown flag bit
    assert L.emu_tcec_gemm_batched(*g, 32, 0) == 1           # FP16 kblock below the 64-k stage
    assert L.emu_tcec_gemm_batched(*g, 96, 0) == 1           # not a multiple of 64
    assert L.emu_tcec_gemm_batched(*g, 0, 8) == 1
    bad = list(g)
    bad[5] = 7                                                 # lda < m
    assert L.emu_tcec_gemm_batched(*bad, 0, 0) == 1
    empty = list(g)
    empty[14] = 0
    assert L.emu_tcec_gemm_batched(*empty, 0, 3) == 0        # batch 0: quick return, flags valid
    # Householder / Givens / scan
    assert L.emu_tcec_householder_batched(8, 8, 16, 8, 16, 7, 64, 16, 8, 64, 1, 0, None, 0) == 1   # ldx < m
    assert L.emu_tcec_householder_batched(8, 8, None, 8, 16, 8, 64, 16, 8, 64, 1, 0, None, 0) == 1
    assert L.emu_tcec_givens_batched(8, 8, 3, 3, 16, 16, 8, 64, 16, 8, 64, 1, 0, None, 0) == 1      # i == j
    assert L.emu_tcec_givens_batched(8, 8, 3, 8, 16, 16, 8, 64, 16, 8, 64, 1, 0, None, 0) == 1      # j >= m
    assert L.emu_tcec_givens_batched(8, 8, 1, 2, 16, 16, 8, 64, 16, 8, 64, 0, 0, None, 0) == 0      # batch 0
    assert L.emu_tcec_scan(8, 4, 16, 7, 16, 8, 0, None, 0) == 1                                    # ldx < n
    assert L.emu_tcec_scan(8, 4, 16, 8, 16, 8, 3, None, 0) == 1                                    # mode
    assert L.emu_tcec_scan(0, 4, None, 1, None, 1, 0, None, 0) == 0                                # n = 0


def test_multicast_validation(emu):
    L = emu.lib
    import ctypes as ct
    arr = (ct.c_void_p * 2)(16, 32)
    assert L.emu_sgemm_multicast(8, 8, 8, 1.0, 16, 8, 16, 8, arr, 0, 8, 0, None, 0, 0) == 1   # num_dst 0
    assert L.emu_sgemm_multicast(8, 8, 8, 1.0, 16, 8, 16, 8, arr, 9, 8, 0, None, 0, 0) == 1   # > 8
    assert L.emu_sgemm_multicast(8, 8, 8, 1.0, 16, 8, 16, 8, None, 1, 8, 0, None, 0, 0) == 1
    bad = (ct.c_void_p * 2)(16, None)
    assert L.emu_sgemm_multicast(8, 8, 8, 1.0, 16, 8, 16, 8, bad, 2, 8, 0, None, 0, 0) == 1
    assert L.emu_sgemm_multicast(-1, 8, 8, 1.0, 16, 8, 16, 8, arr, 2, 8, 0, None, 0, 0) == 1


def test_layout_entry_validation(emu):
    L = emu.lib
    args = [b"N", b"N", 8, 16, 32, 1.0, 16, 32, 0, 16, 16, 0, 0.0, 16, 16, 0, 1, 0, None, None, 0, 0]
    assert L.emu_sgemm_batched_layout(2, *args) == 1                 # unknown layout
    bad = list(args)
    bad[7] = 31                                                      # row-major 'N' A: lda >= k = 32
    assert L.emu_sgemm_batched_layout(1, *bad) == 1
    bad = list(args)
    bad[14] = 15                                                     # row-major C: ldc >= n = 16
    assert L.emu_sgemm_batched_layout(1, *bad) == 1
    assert L.emu_sgemm_batched_layout(1, b"X", b"N", *args[2:]) == 1
    empty = list(args)
    empty[16] = 0                                                    # batch 0
    assert L.emu_sgemm_batched_layout(1, *empty) == 0
