"""CPU-side checks of the C-ABI boundary (no GPU compute): liboqr.so builds for sm_100a, loads,
exports every symbol include/oqr.h declares, validates arguments with the documented negative
status codes before touching the device, and the product path never imports the oracle."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "oqr.h")


@pytest.fixture(scope="module")
def L():
    from paper_1401_5171_b200 import build
    build.build()
    import paper_1401_5171_b200 as oqr
    return oqr.lib()


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(oqr_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ("oqr_normal", "oqr_normal2", "oqr_prequr", "oqr_gram", "oqr_gram_euclid",
              "oqr_potrf", "oqr_trsm", "oqr_status_string"):
        assert s in syms


def test_library_exports_every_declared_symbol(L):
    import paper_1401_5171_b200 as oqr
    syms = declared_symbols()
    assert sorted(oqr.EXPORTS) == syms
    for s in syms:
        assert hasattr(L, s), s
    out = subprocess.run(["nm", "-D", "--defined-only", oqr.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (oqr_[a-z0-9_]+)\b", out))
    assert set(syms) <= exported


def test_library_is_sm100a_only(L):
    import paper_1401_5171_b200 as oqr
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", oqr.LIB_PATH],
                         capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_sass_uses_fp64_tensor_pipe_and_bulk_copy(L):
    import paper_1401_5171_b200 as oqr
    syms = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-symbols", oqr.LIB_PATH],
                          capture_output=True, text=True).stdout
    name = re.search(r"(_ZN3oqr17gram_fused_kernelILi25ELb0EE\w+)", syms).group(1)
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", "-fun", name, oqr.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "DMMA" in out            # mma.sync f64 -> FP64 tensor pipe
    assert "UBLKCP" in out          # cp.async.bulk (packed Z block) -> bulk-copy engine
    assert "UTMALDG" in out         # cp.async.bulk.tensor (A tile) -> tensor TMA


@pytest.mark.parametrize("args,expect", [
    # m, n, A, lda, Z, ldz, Q, R
    ((0, 1, 16, 2, 16, 1, 16, 16), -1),
    ((10, 0, 16, 10, 16, 10, 16, 16), -2),
    ((10, 11, 16, 10, 16, 10, 16, 16), -2),
    ((300, 241, 16, 300, 16, 300, 16, 16), -2),
    ((10, 2, 0, 10, 16, 10, 16, 16), -3),
    ((10, 2, 4, 10, 16, 10, 16, 16), -3),     # A not 8-byte aligned
    ((10, 2, 16, 9, 16, 10, 16, 16), -4),     # lda < m
    ((10, 2, 16, 10, 0, 10, 16, 16), -5),
    ((10, 2, 16, 10, 16, 9, 16, 16), -6),
    ((10, 2, 16, 10, 16, 10, 0, 16), -7),
    ((10, 2, 16, 10, 16, 10, 12, 16), -7),    # Q not 8-byte aligned
    ((10, 2, 16, 10, 16, 10, 16, 0), -8),
])
@pytest.mark.parametrize("fn", ["oqr_normal", "oqr_normal2", "oqr_prequr"])
def test_argument_errors_before_any_device_work(L, fn, args, expect):
    m, n, A, lda, Z, ldz, Q, R = args
    P = ctypes.c_void_p
    st = getattr(L, fn)(m, n, P(A or None), lda, P(Z or None), ldz, P(Q or None), P(R or None), None)
    assert st == expect
    assert L.oqr_status_string(st).decode().startswith(f"invalid argument {-expect}")


def test_status_strings(L):
    assert L.oqr_status_string(0) == b"success"
    assert b"breakdown" in L.oqr_status_string(3)
    assert L.oqr_status_string(-100) == b"CUDA error"


def test_product_path_never_touches_oracle():
    pkg = os.path.join(ROOT, "paper_1401_5171_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in src and "from oracle" not in src, f
                assert "oqr_oracle" not in src and "orc_" not in src, f


def test_fast_path_query_without_gpu():
    """oqr_gram_fast_path is pure host logic (no CUDA call): fast for a 16-byte aligned A with even
    lda, slow for odd lda or an 8-byte offset, argument errors as documented in include/oqr.h."""
    import ctypes
    import paper_1401_5171_b200 as oqr
    L = oqr.lib()
    buf = (ctypes.c_double * 64)()
    base = ctypes.addressof(buf)
    a16 = base + ((-base) % 16)
    assert L.oqr_gram_fast_path(4, ctypes.c_void_p(a16), 4) == 1
    assert L.oqr_gram_fast_path(4, ctypes.c_void_p(a16), 5) == 0
    assert L.oqr_gram_fast_path(4, ctypes.c_void_p(a16 + 8), 4) == 0
    assert L.oqr_gram_fast_path(4, ctypes.c_void_p(a16 + 4), 4) == -3
    assert L.oqr_gram_fast_path(4, None, 4) == -3
    assert L.oqr_gram_fast_path(4, ctypes.c_void_p(a16), 3) == -4
    assert L.oqr_gram_fast_path(0, ctypes.c_void_p(a16), 4) == -1
