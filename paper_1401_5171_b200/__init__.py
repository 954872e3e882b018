"""Thin Python binding of liboqr.so (B200 / sm_100a oblique QR, normal-equation path).

Argument marshalling only: every arithmetic step runs in the library's CUDA kernels (see
``include/oqr.h`` for the contract and PAPER.md citations).  PyTorch supplies device memory
and the stream.  There is no CPU fallback: if ``liboqr.so`` is missing or no CUDA device is
present, calls raise.

Layout: a column-major ``rows x cols`` matrix with leading dimension ``ld`` is a C-contiguous
float64 tensor of shape ``(cols, ld)`` (element (i, j) is ``t[j, i]``) -- the same convention as
``gen`` and the CPU checker.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# OQR_LIB overrides the library path (experiment builds under tools/exp only).
LIB_PATH = os.environ.get("OQR_LIB") or os.path.join(_HERE, "liboqr.so")
NMAX = 240

__all__ = ["normal", "normal2", "prequr", "gram", "gram_euclid", "potrf", "trsm", "status_string",
           "OqrError", "lib", "LIB_PATH", "NMAX", "timing_enable", "timing_reset", "timing_read",
           "launch_count", "EXPORTS", "normal_host"]

# Every symbol include/oqr.h declares.
EXPORTS = ("oqr_normal", "oqr_normal_host", "oqr_normal2", "oqr_prequr", "oqr_workspace_bytes", "oqr_normal_async",
           "oqr_normal2_async", "oqr_prequr_async", "oqr_prequr_stable_async", "oqr_prequr_stable", "oqr_prequr_stable_sym",
           "oqr_prequr_hh", "oqr_prequr_hh_sym", "oqr_prequr_hh_tridiag", "oqr_prequr_hh_async", "oqr_hhqr",
           "oqr_prequr_stable_tridiag", "oqr_normal_sym", "oqr_normal2_sym", "oqr_prequr_sym",
           "oqr_gram_sym", "oqr_upload_sym", "oqr_normal_tridiag", "oqr_normal2_tridiag",
           "oqr_prequr_tridiag", "oqr_gram_tridiag", "oqr_status_string", "oqr_gram",
           "oqr_gram_euclid", "oqr_potrf", "oqr_trsm", "oqr_trmm", "oqr_gram_rows", "oqr_sum_partials",
           "oqr_timing_enable", "oqr_timing_reset", "oqr_timing_read", "oqr_timing_read_kernel",
           "oqr_launch_count", "oqr_pool_trim", "oqr_pool_reserved", "oqr_gram_fast_path")


class OqrError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        super().__init__(f"{where}: status {status}: {status_string(status)}")


_lib = None


def lib() -> ctypes.CDLL:
    """Load liboqr.so (raises if it has not been built -- there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: build it with "
                               "`python -c 'import __graft_entry__ as g; g.build()'`")
        L = ctypes.CDLL(LIB_PATH)
        I64, P, I = ctypes.c_int64, ctypes.c_void_p, ctypes.c_int
        for name in ("oqr_normal", "oqr_normal2", "oqr_prequr", "oqr_normal_sym", "oqr_normal2_sym",
                     "oqr_prequr_sym", "oqr_prequr_stable", "oqr_prequr_stable_sym", "oqr_prequr_hh",
                     "oqr_prequr_hh_sym"):
            f = getattr(L, name)
            f.restype = I
            f.argtypes = [I64, I64, P, I64, P, I64, P, P, P]
        for name in ("oqr_normal_tridiag", "oqr_normal2_tridiag", "oqr_prequr_tridiag", "oqr_prequr_stable_tridiag",
                     "oqr_prequr_hh_tridiag"):
            f = getattr(L, name)
            f.restype = I
            f.argtypes = [I64, I64, P, P, P, I64, P, P, P]
        L.oqr_gram_tridiag.restype = I
        L.oqr_gram_tridiag.argtypes = [I64, I64, P, P, P, I64, P, P]
        L.oqr_status_string.restype = ctypes.c_char_p
        L.oqr_status_string.argtypes = [I]
        L.oqr_workspace_bytes.restype = ctypes.c_size_t
        L.oqr_workspace_bytes.argtypes = [I64, I64]
        for name in ("oqr_normal_async", "oqr_normal2_async", "oqr_prequr_async", "oqr_prequr_stable_async",
                     "oqr_prequr_hh_async"):
            f = getattr(L, name)
            f.restype = I
            f.argtypes = [I64, I64, P, I64, P, I64, P, P, P, ctypes.c_size_t, P, P]
        L.oqr_normal_host.restype = I
        L.oqr_normal_host.argtypes = [I64, I64, P, I64, P, I64, P, P, I64, P]
        L.oqr_upload_sym.restype = I
        L.oqr_upload_sym.argtypes = [I64, P, I64, P, I64, P]
        L.oqr_gram_sym.restype = I
        L.oqr_gram_sym.argtypes = [I64, I64, P, I64, P, I64, P, P]
        L.oqr_gram.restype = I
        L.oqr_gram.argtypes = [I64, I64, P, I64, P, I64, P, P]
        L.oqr_gram_euclid.restype = I
        L.oqr_gram_euclid.argtypes = [I64, I64, P, I64, P, P]
        L.oqr_potrf.restype = I
        L.oqr_potrf.argtypes = [I64, P, P, P, P]
        L.oqr_trsm.restype = I
        L.oqr_trsm.argtypes = [I64, I64, P, I64, P, P, P]
        L.oqr_trmm.restype = I
        L.oqr_trmm.argtypes = [I64, P, P, P, P]
        L.oqr_hhqr.restype = I
        L.oqr_hhqr.argtypes = [I64, I64, P, I64, P, P, P]
        L.oqr_gram_rows.restype = I
        L.oqr_gram_rows.argtypes = [I64, I64, I64, I64, P, I64, P, I64, P, P]
        L.oqr_sum_partials.restype = I
        L.oqr_sum_partials.argtypes = [I64, I64, P, P, P]
        L.oqr_timing_enable.restype = None
        L.oqr_timing_enable.argtypes = [I]
        L.oqr_timing_reset.restype = None
        L.oqr_timing_reset.argtypes = []
        L.oqr_timing_read.restype = I
        L.oqr_timing_read.argtypes = [ctypes.POINTER(ctypes.c_double), ctypes.POINTER(I64),
                                      ctypes.POINTER(I64)]
        L.oqr_timing_read_kernel.restype = I
        L.oqr_timing_read_kernel.argtypes = [I, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(I64)]
        L.oqr_gram_fast_path.restype = I
        L.oqr_gram_fast_path.argtypes = [I64, P, I64]
        L.oqr_pool_trim.restype = I
        L.oqr_pool_trim.argtypes = [ctypes.c_size_t]
        L.oqr_pool_reserved.restype = I64
        L.oqr_pool_reserved.argtypes = []
        L.oqr_launch_count.restype = I64
        L.oqr_launch_count.argtypes = []
        _lib = L
    return _lib


def status_string(status: int) -> str:
    return lib().oqr_status_string(int(status)).decode()


def _stream(stream):
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def _check(t, name: str, rows: int | None = None):
    import torch
    if not isinstance(t, torch.Tensor) or t.dtype != torch.float64 or not t.is_cuda:
        raise TypeError(f"{name}: expected a float64 CUDA tensor")
    if t.dim() != 2 or not t.is_contiguous():
        raise TypeError(f"{name}: expected a contiguous 2-D tensor of shape (cols, ld)")
    if rows is not None and t.shape[1] < rows:
        raise ValueError(f"{name}: leading dimension {t.shape[1]} < {rows}")
    return ctypes.c_void_p(t.data_ptr())


def _variant(fname: str, A, Z, Q=None, R=None, stream=None, check: bool = True):
    import torch
    m = A.shape[0]
    n = Z.shape[0]
    pA = _check(A, "A", m)
    pZ = _check(Z, "Z", m)
    if Q is None:
        Q = torch.empty((n, m), dtype=torch.float64, device=Z.device)
    if R is None:
        R = torch.empty((n, n), dtype=torch.float64, device=Z.device)
    pQ = _check(Q, "Q", m)
    pR = _check(R, "R", n)
    if Q.shape != (n, m) or R.shape != (n, n):
        raise ValueError("Q must be (n, m) and R (n, n)")
    st = getattr(lib(), fname)(m, n, pA, A.shape[1], pZ, Z.shape[1], pQ, pR, _stream(stream))
    if check and st < 0:
        raise OqrError(st, fname)
    return Q, R, st


def normal(A, Z, Q=None, R=None, stream=None, check: bool = True):
    """CHOLQR, Algorithm 1.  Returns (Q, R, status); status > 0 is a
    Cholesky breakdown (see include/oqr.h), negative statuses raise unless check=False."""
    return _variant("oqr_normal", A, Z, Q, R, stream, check)


def _host(t, name: str, rows: int):
    import torch
    if not isinstance(t, torch.Tensor) or t.dtype != torch.float64 or t.is_cuda:
        raise TypeError(f"{name}: expected a float64 CPU tensor")
    if t.dim() != 2 or not t.is_contiguous():
        raise TypeError(f"{name}: expected a contiguous 2-D tensor of shape (cols, ld)")
    if t.shape[1] < rows:
        raise ValueError(f"{name}: leading dimension {t.shape[1]} < {rows}")
    return ctypes.c_void_p(t.data_ptr())


def normal_host(A, Z, Q=None, R=None, chunk_cols: int = 0, stream=None, check: bool = True):
    """oqr_normal on HOST tensors (pinned for full PCIe bandwidth and copy/compute overlap):
    A is staged to the device in column chunks while the fused Gram runs on the chunks already
    there (include/oqr.h).  Returns host (Q, R, status)."""
    import torch
    m, n = A.shape[0], Z.shape[0]
    pin = A.is_pinned()
    if Q is None:
        Q = torch.empty((n, m), dtype=torch.float64, pin_memory=pin)
    if R is None:
        R = torch.empty((n, n), dtype=torch.float64, pin_memory=pin)
    if Q.shape != (n, m) or R.shape != (n, n):
        raise ValueError("Q must be (n, m) and R (n, n)")
    st = lib().oqr_normal_host(m, n, _host(A, "A", m), A.shape[1], _host(Z, "Z", m), Z.shape[1], _host(Q, "Q", m),
                               _host(R, "R", n), int(chunk_cols), _stream(stream))
    if check and st < 0:
        raise OqrError(st, "oqr_normal_host")
    return Q, R, st


def normal2(A, Z, Q=None, R=None, stream=None, check: bool = True):
    """Repeated CHOLQR: two passes, R = R2 R1 (reading R1)."""
    return _variant("oqr_normal2", A, Z, Q, R, stream, check)


def prequr(A, Z, Q=None, R=None, stream=None, check: bool = True):
    """PRE-CHOLQR, Algorithm 2 with a Euclidean Cholesky-QR pre-step."""
    return _variant("oqr_prequr", A, Z, Q, R, stream, check)


def prequr_stable(A, Z, Q=None, R=None, stream=None, check: bool = True):
    """PRE-CHOLQR with the stable shifted-CholeskyQR3 Euclidean pre-step (NEXT-N1, reading R21)."""
    return _variant("oqr_prequr_stable", A, Z, Q, R, stream, check)


def prequr_hh(A, Z, Q=None, R=None, stream=None, check: bool = True):
    """PRE-CHOLQR exactly as Algorithm 2 states it: Householder QR pre-step (NEXT-N1, paper-faithful)."""
    return _variant("oqr_prequr_hh", A, Z, Q, R, stream, check)


VARIANTS = {"normal": normal, "normal2": normal2, "prequr": prequr, "prequr_stable": prequr_stable,
            "prequr_hh": prequr_hh}


def normal_sym(A, Z, Q=None, R=None, stream=None, check: bool = True):
    """CHOLQR reading only the block-lower triangle of the (symmetric) A (NEXT-N4)."""
    return _variant("oqr_normal_sym", A, Z, Q, R, stream, check)


def normal2_sym(A, Z, Q=None, R=None, stream=None, check: bool = True):
    return _variant("oqr_normal2_sym", A, Z, Q, R, stream, check)


def prequr_sym(A, Z, Q=None, R=None, stream=None, check: bool = True):
    return _variant("oqr_prequr_sym", A, Z, Q, R, stream, check)


def prequr_stable_sym(A, Z, Q=None, R=None, stream=None, check: bool = True):
    return _variant("oqr_prequr_stable_sym", A, Z, Q, R, stream, check)


def prequr_hh_sym(A, Z, Q=None, R=None, stream=None, check: bool = True):
    return _variant("oqr_prequr_hh_sym", A, Z, Q, R, stream, check)


VARIANTS_SYM = {"normal": normal_sym, "normal2": normal2_sym, "prequr": prequr_sym, "prequr_stable": prequr_stable_sym,
                "prequr_hh": prequr_hh_sym}


def upload_sym(A_host, A_dev, stream=None):
    """Copy the block-lower triangle of a (pinned) host A into A_dev: what the *_sym calls read."""
    import torch
    if A_host.is_cuda or A_host.dtype != torch.float64 or not A_host.is_contiguous():
        raise TypeError("A_host: expected a contiguous float64 CPU tensor (m, lda)")
    m = A_host.shape[0]
    st = lib().oqr_upload_sym(m, ctypes.c_void_p(A_host.data_ptr()), A_host.shape[1], _check(A_dev, "A_dev", m),
                              A_dev.shape[1], _stream(stream))
    if st:
        raise OqrError(st, "oqr_upload_sym")
    return A_dev


def gram_sym(A, Z, G=None, stream=None):
    """Symmetric Gram G = T + T^T from the block-lower triangle of A (asynchronous step export)."""
    import torch
    m, n = A.shape[0], Z.shape[0]
    if G is None:
        G = torch.empty((n, n), dtype=torch.float64, device=Z.device)
    st = lib().oqr_gram_sym(m, n, _check(A, "A", m), A.shape[1], _check(Z, "Z", m), Z.shape[1],
                            _check(G, "G", n), _stream(stream))
    if st:
        raise OqrError(st, "oqr_gram_sym")
    return G


def _vec(t, name: str, length: int):
    import torch
    if not isinstance(t, torch.Tensor) or t.dtype != torch.float64 or not t.is_cuda or t.dim() != 1:
        raise TypeError(f"{name}: expected a 1-D float64 CUDA tensor")
    if t.numel() < length or not t.is_contiguous():
        raise ValueError(f"{name}: expected {length} contiguous entries")
    return ctypes.c_void_p(t.data_ptr()) if length > 0 else ctypes.c_void_p(None)


def _variant_tridiag(fname: str, d, e, Z, Q=None, R=None, stream=None, check: bool = True):
    import torch
    m, n = d.numel(), Z.shape[0]
    pd, pe = _vec(d, "d", m), _vec(e, "e", m - 1)
    pZ = _check(Z, "Z", m)
    if Q is None:
        Q = torch.empty((n, m), dtype=torch.float64, device=Z.device)
    if R is None:
        R = torch.empty((n, n), dtype=torch.float64, device=Z.device)
    st = getattr(lib(), fname)(m, n, pd, pe, pZ, Z.shape[1], _check(Q, "Q", m), _check(R, "R", n), _stream(stream))
    if check and st < 0:
        raise OqrError(st, fname)
    return Q, R, st


def normal_tridiag(d, e, Z, Q=None, R=None, stream=None, check: bool = True):
    """CHOLQR with tridiagonal A = tridiag(e, d, e) (NEXT-N3)."""
    return _variant_tridiag("oqr_normal_tridiag", d, e, Z, Q, R, stream, check)


def normal2_tridiag(d, e, Z, Q=None, R=None, stream=None, check: bool = True):
    return _variant_tridiag("oqr_normal2_tridiag", d, e, Z, Q, R, stream, check)


def prequr_tridiag(d, e, Z, Q=None, R=None, stream=None, check: bool = True):
    return _variant_tridiag("oqr_prequr_tridiag", d, e, Z, Q, R, stream, check)


def prequr_stable_tridiag(d, e, Z, Q=None, R=None, stream=None, check: bool = True):
    return _variant_tridiag("oqr_prequr_stable_tridiag", d, e, Z, Q, R, stream, check)


def prequr_hh_tridiag(d, e, Z, Q=None, R=None, stream=None, check: bool = True):
    return _variant_tridiag("oqr_prequr_hh_tridiag", d, e, Z, Q, R, stream, check)


VARIANTS_TRIDIAG = {"normal": normal_tridiag, "normal2": normal2_tridiag, "prequr": prequr_tridiag,
                    "prequr_stable": prequr_stable_tridiag, "prequr_hh": prequr_hh_tridiag}


def gram_tridiag(d, e, Z, G=None, stream=None):
    """G = Z^T (T Z) for T = tridiag(e, d, e) (asynchronous step export)."""
    import torch
    m, n = d.numel(), Z.shape[0]
    if G is None:
        G = torch.empty((n, n), dtype=torch.float64, device=Z.device)
    st = lib().oqr_gram_tridiag(m, n, _vec(d, "d", m), _vec(e, "e", m - 1), _check(Z, "Z", m), Z.shape[1],
                                _check(G, "G", n), _stream(stream))
    if st:
        raise OqrError(st, "oqr_gram_tridiag")
    return G


def gram(A, Z, G=None, stream=None):
    """G = Z^T (A Z) (asynchronous step export).  Returns G as a (n, n) column-major tensor."""
    import torch
    m, n = A.shape[0], Z.shape[0]
    if G is None:
        G = torch.empty((n, n), dtype=torch.float64, device=Z.device)
    st = lib().oqr_gram(m, n, _check(A, "A", m), A.shape[1], _check(Z, "Z", m), Z.shape[1],
                        _check(G, "G", n), _stream(stream))
    if st:
        raise OqrError(st, "oqr_gram")
    return G


def gram_euclid(Z, m: int | None = None, G=None, stream=None):
    """G = Z^T Z (asynchronous step export)."""
    import torch
    n = Z.shape[0]
    m = Z.shape[1] if m is None else m
    if G is None:
        G = torch.empty((n, n), dtype=torch.float64, device=Z.device)
    st = lib().oqr_gram_euclid(m, n, _check(Z, "Z", m), Z.shape[1], _check(G, "G", n), _stream(stream))
    if st:
        raise OqrError(st, "oqr_gram_euclid")
    return G


def potrf(G, R=None, info=None, stream=None):
    """R = chol(G) (upper); returns (R, info tensor (1,) int32 on device)."""
    import torch
    n = G.shape[0]
    if R is None:
        R = torch.empty((n, n), dtype=torch.float64, device=G.device)
    if info is None:
        info = torch.zeros(1, dtype=torch.int32, device=G.device)
    st = lib().oqr_potrf(n, _check(G, "G", n), _check(R, "R", n), ctypes.c_void_p(info.data_ptr()),
                         _stream(stream))
    if st:
        raise OqrError(st, "oqr_potrf")
    return R, info


def trsm(Z, R, m: int | None = None, Q=None, stream=None):
    """Q = Z R^{-1} by row-wise substitution (asynchronous step export)."""
    import torch
    n = Z.shape[0]
    m = Z.shape[1] if m is None else m
    if Q is None:
        Q = torch.empty((n, m), dtype=torch.float64, device=Z.device)
    st = lib().oqr_trsm(m, n, _check(Z, "Z", m), Z.shape[1], _check(R, "R", n), _check(Q, "Q", m),
                        _stream(stream))
    if st:
        raise OqrError(st, "oqr_trsm")
    return Q


def hhqr(Z, m: int | None = None, Y=None, S=None, stream=None):
    """[Y, S] = Householder QR of Z, positive-diagonal S (asynchronous step export of K6)."""
    import torch
    n = Z.shape[0]
    m = Z.shape[1] if m is None else m
    if Y is None:
        Y = torch.empty((n, m), dtype=torch.float64, device=Z.device)
    if S is None:
        S = torch.empty((n, n), dtype=torch.float64, device=Z.device)
    st = lib().oqr_hhqr(m, n, _check(Z, "Z", m), Z.shape[1], _check(Y, "Y", m), _check(S, "S", n), _stream(stream))
    if st:
        raise OqrError(st, "oqr_hhqr")
    return Y, S


def gram_rows(Ar, Z, r0: int, mr: int, G=None, stream=None):
    """Partial Gram of a row shard: Z_R^T (A_{R,:} Z), R = [r0, r0 + mr).  Ar: (m, ldar) tensor
    holding the mr x m row block column-major (ldar >= mr); Z: (n, ldz) with all m rows."""
    import torch
    n, m = Z.shape[0], Ar.shape[0]
    if G is None:
        G = torch.empty((n, n), dtype=torch.float64, device=Z.device)
    st = lib().oqr_gram_rows(m, n, r0, mr, _check(Ar, "Ar", mr), Ar.shape[1], _check(Z, "Z", m), Z.shape[1],
                             _check(G, "G", n), _stream(stream))
    if st:
        raise OqrError(st, "oqr_gram_rows")
    return G


def sum_partials(P, G=None, stream=None):
    """G = sum_c P[c] in c order; P: (count, n, n) tensor of column-major n x n partials."""
    import torch
    count, n = P.shape[0], P.shape[1]
    if not P.is_contiguous() or P.dtype != torch.float64 or not P.is_cuda:
        raise TypeError("P: expected a contiguous float64 CUDA tensor (count, n, n)")
    if G is None:
        G = torch.empty((n, n), dtype=torch.float64, device=P.device)
    st = lib().oqr_sum_partials(n, count, ctypes.c_void_p(P.data_ptr()), _check(G, "G", n), _stream(stream))
    if st:
        raise OqrError(st, "oqr_sum_partials")
    return G


def trsm_rows(Z, R, r0: int, mr: int, Q=None, stream=None):
    """Q_local = Z[r0:r0+mr, :] R^{-1} (rows of a shard); Z: (n, ldz) with all rows; Q: (n, mr)."""
    import torch
    n = Z.shape[0]
    if Q is None:
        Q = torch.empty((n, mr), dtype=torch.float64, device=Z.device)
    _check(Z, "Z", r0 + mr)
    zp = ctypes.c_void_p(Z.data_ptr() + 8 * r0)
    st = lib().oqr_trsm(mr, n, zp, Z.shape[1], _check(R, "R", n), _check(Q, "Q", mr), _stream(stream))
    if st:
        raise OqrError(st, "oqr_trsm")
    return Q


def gram_euclid_rows(Z, r0: int, mr: int, G=None, stream=None):
    """G_r = Z_R^T Z_R for the rows R = [r0, r0 + mr) of Z (n, ldz) (asynchronous)."""
    import torch
    n = Z.shape[0]
    if G is None:
        G = torch.empty((n, n), dtype=torch.float64, device=Z.device)
    _check(Z, "Z", r0 + mr)
    st = lib().oqr_gram_euclid(mr, n, ctypes.c_void_p(Z.data_ptr() + 8 * r0), Z.shape[1], _check(G, "G", n),
                               _stream(stream))
    if st:
        raise OqrError(st, "oqr_gram_euclid")
    return G


def trmm(R2, R1, R=None, stream=None):
    """R = R2 R1 for upper triangular (n, n) tensors (asynchronous step export)."""
    import torch
    n = R1.shape[0]
    if R is None:
        R = torch.empty((n, n), dtype=torch.float64, device=R1.device)
    st = lib().oqr_trmm(n, _check(R2, "R2", n), _check(R1, "R1", n), _check(R, "R", n), _stream(stream))
    if st:
        raise OqrError(st, "oqr_trmm")
    return R


def workspace_bytes(m: int, n: int) -> int:
    """Bytes of caller workspace the *_async calls need (upper bound over all variants)."""
    return int(lib().oqr_workspace_bytes(m, n))


def _async(fname: str, A, Z, Q, R, workspace, status, stream=None):
    m, n = A.shape[0], Z.shape[0]
    ws = ctypes.c_void_p(workspace.data_ptr()) if workspace is not None else ctypes.c_void_p(None)
    wsb = workspace.numel() * workspace.element_size() if workspace is not None else 0
    st = getattr(lib(), fname)(m, n, _check(A, "A", m), A.shape[1], _check(Z, "Z", m), Z.shape[1],
                               _check(Q, "Q", m), _check(R, "R", n), ws, wsb, ctypes.c_void_p(status.data_ptr()),
                               _stream(stream))
    if st:
        raise OqrError(st, fname)


def normal_async(A, Z, Q, R, workspace, status, stream=None):
    """Enqueue CHOLQR without synchronising (CUDA-graph capturable with a workspace tensor of
    workspace_bytes(m, n) bytes); the factorisation status lands in `status` (int32 CUDA tensor)."""
    _async("oqr_normal_async", A, Z, Q, R, workspace, status, stream)


def normal2_async(A, Z, Q, R, workspace, status, stream=None):
    _async("oqr_normal2_async", A, Z, Q, R, workspace, status, stream)


def prequr_async(A, Z, Q, R, workspace, status, stream=None):
    _async("oqr_prequr_async", A, Z, Q, R, workspace, status, stream)


def prequr_stable_async(A, Z, Q, R, workspace, status, stream=None):
    _async("oqr_prequr_stable_async", A, Z, Q, R, workspace, status, stream)


def prequr_hh_async(A, Z, Q, R, workspace, status, stream=None):
    _async("oqr_prequr_hh_async", A, Z, Q, R, workspace, status, stream)


VARIANTS_ASYNC = {"normal": normal_async, "normal2": normal2_async, "prequr": prequr_async,
                  "prequr_stable": prequr_stable_async, "prequr_hh": prequr_hh_async}


def timing_enable(on: bool = True):
    lib().oqr_timing_enable(1 if on else 0)


def timing_reset():
    lib().oqr_timing_reset()


TIMING_KERNELS = {"K1": 0, "K4": 1, "K3": 2, "K2": 3, "K6": 4}


def timing_read_kernel(kernel: str) -> tuple[float, int]:
    """(accumulated milliseconds, launches) of one kernel family ("K1" fused Gram, "K4" packed
    Gram, "K3" triangular solve, "K2" Cholesky) since the last timing_reset."""
    ms = ctypes.c_double()
    k = ctypes.c_int64()
    st = lib().oqr_timing_read_kernel(TIMING_KERNELS[kernel], ctypes.byref(ms), ctypes.byref(k))
    if st:
        raise OqrError(st, "oqr_timing_read_kernel")
    return ms.value, k.value


def timing_read() -> tuple[float, int, int]:
    """(accumulated K1 milliseconds, K1 launches, all library launches) since the last reset."""
    ms = ctypes.c_double()
    k1 = ctypes.c_int64()
    tot = ctypes.c_int64()
    st = lib().oqr_timing_read(ctypes.byref(ms), ctypes.byref(k1), ctypes.byref(tot))
    if st:
        raise OqrError(st, "oqr_timing_read")
    return ms.value, k1.value, tot.value


def gram_fast_path(A) -> bool:
    """True when the fused Gram kernel reads this A (tensor (m, lda)) through tensor TMA (16-byte
    aligned, even lda); False for the plain-load slow path."""
    m = A.shape[0]
    st = lib().oqr_gram_fast_path(m, _check(A, "A", m), A.shape[1])
    if st < 0:
        raise OqrError(st, "oqr_gram_fast_path")
    return st == 1


def pool_trim(keep_bytes: int = 0) -> None:
    """Release the library pool's cached device memory down to keep_bytes (synchronises the device)."""
    st = lib().oqr_pool_trim(int(keep_bytes))
    if st:
        raise OqrError(st, "oqr_pool_trim")


def pool_reserved() -> int:
    """Bytes of device memory the library pool currently holds."""
    return int(lib().oqr_pool_reserved())


def launch_count() -> int:
    return int(lib().oqr_launch_count())
