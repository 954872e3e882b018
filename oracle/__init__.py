"""CPU FP64 oracle for the oblique-QR normal-equation path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` leg may import this package.  The product path
(``paper_1401_5171_b200``) never imports it and shares no code with it.

The arithmetic lives in ``oqr_oracle.c`` (plain C, FP64, no FMA contraction; see its header
for the PAPER.md citations of every routine).  This module only marshals numpy arrays and
adds the norm helpers used by the gates (LAPACK SVD / eigvalsh as library primitives).

Layout: a column-major ``rows x cols`` matrix with leading dimension ``ld`` is a C-contiguous
numpy array of shape ``(cols, ld)``.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboqr_oracle.so")
U = 2.0 ** -53  # unit roundoff


def gamma(k: float) -> float:
    """gamma_k = k u / (1 - k u) (Higham; the paper's c*k*u with c = 1)."""
    return k * U / (1.0 - k * U)


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "oqr_oracle.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        cmd = (f"gcc -O3 -mavx2 -ffp-contract=off -fno-fast-math -fopenmp -fPIC -shared -Wall "
               f"-o {_LIB_PATH} {src} -lm")
        if os.system(cmd) != 0:
            raise RuntimeError("failed to build oracle/liboqr_oracle.so: " + cmd)
    return _LIB_PATH


_lib = None


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB_PATH)
        I, P = ctypes.c_int64, ctypes.c_void_p
        sig = {
            "orc_gram": (None, [I, I, P, I, P, I, P, I]),
            "orc_gram_euclid": (None, [I, I, P, I, P, I]),
            "orc_potrf": (ctypes.c_int, [I, P, I, P, I]),
            "orc_trsm": (None, [I, I, P, I, P, I, P, I]),
            "orc_trmm": (None, [I, P, I, P, I, P, I]),
            "orc_normal": (ctypes.c_int, [I, I, P, I, P, I, P, P]),
            "orc_normal2": (ctypes.c_int, [I, I, P, I, P, I, P, P]),
            "orc_prequr": (ctypes.c_int, [I, I, P, I, P, I, P, P]),
            "orc_dd_orth": (None, [I, I, P, I, P, I, P]),
            "orc_dd_gram": (None, [I, I, P, I, P, I, P, P]),
            "orc_dd_resid": (None, [I, I, P, I, P, I, P, I, P, P]),
            "orc_dd_chol_resid": (None, [I, P, I, P, I, P, P]),
            "orc_dd_orth_cols": (None, [I, I, P, P, I, P, I, P]),
            "orc_gram_tridiag": (None, [I, I, P, P, P, I, P, I]),
            "orc_scqr3": (ctypes.c_int, [I, I, P, I, P, P]),
            "orc_prequr_stable": (ctypes.c_int, [I, I, P, I, P, I, P, P]),
            "orc_normal_tridiag": (ctypes.c_int, [I, I, P, P, P, I, P, P]),
            "orc_normal2_tridiag": (ctypes.c_int, [I, I, P, P, P, I, P, P]),
            "orc_prequr_tridiag": (ctypes.c_int, [I, I, P, P, P, I, P, P]),
            "orc_dd_orth_tridiag": (None, [I, I, P, P, P, I, P]),
            "orc_geqr2": (None, [I, I, P, I, P]),
            "orc_org2r": (None, [I, I, P, I, P, P]),
            "orc_hhqr": (ctypes.c_int, [I, I, P, I, P, P]),
            "orc_prequr_hh": (ctypes.c_int, [I, I, P, I, P, I, P, P]),
            "orc_dd_orth_euclid": (None, [I, I, P, I, P]),
        }
        for name, (res, args) in sig.items():
            f = getattr(lib, name)
            f.restype = res
            f.argtypes = args
        _lib = lib
    return _lib


def _p(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous, "expected C-contiguous float64"
    return a.ctypes.data_as(ctypes.c_void_p)


def _cm(a: np.ndarray, rows: int) -> tuple[np.ndarray, int]:
    """Return (array, ld) for a column-major matrix stored as (cols, ld)."""
    a = np.ascontiguousarray(a, dtype=np.float64)
    assert a.shape[1] >= rows
    return a, a.shape[1]


def to_cm(M: np.ndarray) -> np.ndarray:
    """Dense row-major numpy matrix (rows x cols) -> column-major storage (cols, rows)."""
    return np.ascontiguousarray(np.asarray(M, dtype=np.float64).T)


def from_cm(a: np.ndarray, rows: int) -> np.ndarray:
    """Column-major storage (cols, ld) -> dense matrix (rows x cols)."""
    return np.ascontiguousarray(a[:, :rows].T)


# ---------------------------------------------------------------- steps ----
def gram(A: np.ndarray, Z: np.ndarray, m: int) -> np.ndarray:
    """G = Z^T (A Z) (Alg. 1 lines 1-2); returns storage (n, n)."""
    A, lda = _cm(A, m)
    Z, ldz = _cm(Z, m)
    n = Z.shape[0]
    G = np.empty((n, n))
    _load().orc_gram(m, n, _p(A), lda, _p(Z), ldz, _p(G), n)
    return G


def gram_euclid(Z: np.ndarray, m: int) -> np.ndarray:
    Z, ldz = _cm(Z, m)
    n = Z.shape[0]
    G = np.empty((n, n))
    _load().orc_gram_euclid(m, n, _p(Z), ldz, _p(G), n)
    return G


def potrf(G: np.ndarray) -> tuple[np.ndarray, int]:
    """Upper Cholesky (Alg. 1 line 3); returns (R storage (n, n), info)."""
    G = np.ascontiguousarray(G, dtype=np.float64)
    n = G.shape[0]
    R = np.empty((n, n))
    info = _load().orc_potrf(n, _p(G), G.shape[1], _p(R), n)
    return R, info


def trsm(Z: np.ndarray, R: np.ndarray, m: int) -> np.ndarray:
    """Q = Z R^{-1} by row-wise substitution (Alg. 1 line 4)."""
    Z, ldz = _cm(Z, m)
    R = np.ascontiguousarray(R, dtype=np.float64)
    n = Z.shape[0]
    Q = np.empty((n, m))
    _load().orc_trsm(m, n, _p(Z), ldz, _p(R), R.shape[1], _p(Q), m)
    return Q


def trmm(R2: np.ndarray, R1: np.ndarray) -> np.ndarray:
    R2 = np.ascontiguousarray(R2, dtype=np.float64)
    R1 = np.ascontiguousarray(R1, dtype=np.float64)
    n = R1.shape[0]
    R = np.empty((n, n))
    _load().orc_trmm(n, _p(R2), R2.shape[1], _p(R1), R1.shape[1], _p(R), n)
    return R


# ------------------------------------------------------------- variants ----
def _variant(fn: str, A: np.ndarray, Z: np.ndarray, m: int):
    A, lda = _cm(A, m)
    Z, ldz = _cm(Z, m)
    n = Z.shape[0]
    Q = np.zeros((n, m))
    R = np.zeros((n, n))
    info = getattr(_load(), fn)(m, n, _p(A), lda, _p(Z), ldz, _p(Q), _p(R))
    return Q, R, info


def normal(A, Z, m):
    """CHOLQR (Alg. 1) -> (Q storage (n, m), R storage (n, n), info)."""
    return _variant("orc_normal", A, Z, m)


def normal2(A, Z, m):
    """Repeated CHOLQR (two passes, R = R2 R1; reading R1)."""
    return _variant("orc_normal2", A, Z, m)


def prequr(A, Z, m):
    """PRE-CHOLQR (Alg. 2) with a Euclidean Cholesky-QR pre-step."""
    return _variant("orc_prequr", A, Z, m)


def prequr_stable(A, Z, m):
    """PRE-CHOLQR with the stable (shifted CholeskyQR3) Euclidean pre-step (NEXT-N1, reading R21)."""
    return _variant("orc_prequr_stable", A, Z, m)


def scqr3(Z, m):
    """Shifted CholeskyQR3 of Z: (Y storage (n, m), S storage (n, n), info)."""
    Z, ldz = _cm(Z, m)
    n = Z.shape[0]
    Y = np.zeros((n, m))
    S = np.zeros((n, n))
    info = _load().orc_scqr3(m, n, _p(Z), ldz, _p(Y), _p(S))
    return Y, S, info


def prequr_hh(A, Z, m):
    """PRE-CHOLQR exactly as Algorithm 2 states it: Householder QR pre-step
    (NEXT-N1, paper-faithful), then CHOLQR(A, Y) and R = U S."""
    return _variant("orc_prequr_hh", A, Z, m)


def hhqr(Z, m):
    """Householder QR of Z with positive-diagonal S: (Y storage (n, m), S storage (n, n))."""
    Z, ldz = _cm(Z, m)
    n = Z.shape[0]
    Y = np.zeros((n, m))
    S = np.zeros((n, n))
    _load().orc_hhqr(m, n, _p(Z), ldz, _p(Y), _p(S))
    return Y, S


def geqr2(Z, m):
    """LAPACK-convention unblocked Householder QR: (X storage (n, m) with R on/above and the
    reflector vectors below the diagonal, tau (n,))."""
    X, ldx = _cm(np.array(Z, dtype=np.float64, copy=True), m)
    n = X.shape[0]
    tau = np.zeros(n)
    _load().orc_geqr2(m, n, _p(X), ldx, _p(tau))
    return X, tau


def orth_error_euclid(Y, m) -> float:
    """||Y^T Y - I||_2, check formed in double-double."""
    Y, ldy = _cm(Y, m)
    n = Y.shape[0]
    E = np.empty((n, n))
    _load().orc_dd_orth_euclid(m, n, _p(Y), ldy, _p(E))
    return float(np.linalg.norm(E.T, 2))


def dd_orth_euclid_matrix(Y, m) -> np.ndarray:
    Y, ldy = _cm(Y, m)
    n = Y.shape[0]
    E = np.empty((n, n))
    _load().orc_dd_orth_euclid(m, n, _p(Y), ldy, _p(E))
    return E.T.copy()


VARIANTS = {"normal": normal, "normal2": normal2, "prequr": prequr, "prequr_stable": prequr_stable,
            "prequr_hh": prequr_hh}


# -------------------------------------------------------------- checkers ---
def dd_orth_matrix(A, Q, m) -> np.ndarray:
    """Q^T A Q - I (double-double accumulation), as a dense n x n matrix."""
    A, lda = _cm(A, m)
    Q, ldq = _cm(Q, m)
    n = Q.shape[0]
    E = np.empty((n, n))
    _load().orc_dd_orth(m, n, _p(A), lda, _p(Q), ldq, _p(E))
    return E.T.copy()


def dd_orth_cols(A, Q, m, cols) -> np.ndarray:
    """Q_S^T A Q_S - I for the column subset S = cols (double-double), dense |S| x |S|.
    Same entries as dd_orth_matrix(A, Q, m)[S][:, S] (sampled checks at full sizes)."""
    A, lda = _cm(A, m)
    Q, ldq = _cm(Q, m)
    c = np.ascontiguousarray(np.asarray(cols, dtype=np.int64))
    ns = len(c)
    E = np.empty((ns, ns))
    _load().orc_dd_orth_cols(m, ns, c.ctypes.data_as(ctypes.c_void_p), _p(A), lda, _p(Q), ldq, _p(E))
    return E.T.copy()


def orth_error(A, Q, m) -> float:
    """||Q^T A Q - I||_2, check formed in double-double."""
    E = dd_orth_matrix(A, Q, m)
    return float(np.linalg.norm(E, 2))


def dd_gram(A, Z, m) -> tuple[np.ndarray, np.ndarray]:
    """(G, M): G = Z^T A Z in double-double (dense n x n), M = |Z|^T |A| |Z|."""
    A, lda = _cm(A, m)
    Z, ldz = _cm(Z, m)
    n = Z.shape[0]
    G = np.empty((n, n))
    M = np.empty((n, n))
    _load().orc_dd_gram(m, n, _p(A), lda, _p(Z), ldz, _p(G), _p(M))
    return G.T.copy(), M.T.copy()


def dd_resid(Z, Q, R, m) -> tuple[np.ndarray, np.ndarray]:
    """(D, QRabs) dense m x n: D = Z - QR (double-double), QRabs = |Q||R|."""
    Z, ldz = _cm(Z, m)
    Q, ldq = _cm(Q, m)
    R = np.ascontiguousarray(R, dtype=np.float64)
    n = Z.shape[0]
    D = np.empty((n, m))
    QR = np.empty((n, m))
    _load().orc_dd_resid(m, n, _p(Z), ldz, _p(Q), ldq, _p(R), R.shape[1], _p(D), _p(QR))
    return D.T.copy(), QR.T.copy()


def componentwise_ratio(Z, Q, R, m) -> float:
    """rho = max_ij |Z - QR|_ij / (|Q||R|)_ij (Theorem 2 componentwise form),
    skipping entries whose denominator is below u * max|Z| (0/0 guard)."""
    D, QR = dd_resid(Z, Q, R, m)
    zmax = float(np.abs(from_cm(np.asarray(Z), m)).max())
    mask = QR > U * zmax
    if not mask.any():
        return 0.0
    return float((np.abs(D)[mask] / QR[mask]).max())


def repr_error(Z, Q, R, m) -> float:
    """||Z - QR||_2 / ||Z||_2, residual formed in double-double."""
    D, _ = dd_resid(Z, Q, R, m)
    return float(np.linalg.norm(D, 2) / np.linalg.norm(from_cm(np.asarray(Z), m), 2))


def chol_backward_ratio(G_dense: np.ndarray, R_store: np.ndarray) -> float:
    """max over the upper triangle of |G - R^T R| / (|R|^T |R|) (eq:normal:chol)."""
    G = to_cm(G_dense)
    R = np.ascontiguousarray(R_store, dtype=np.float64)
    n = G.shape[0]
    D = np.empty((n, n))
    RR = np.empty((n, n))
    _load().orc_dd_chol_resid(n, _p(G), n, _p(R), R.shape[1], _p(D), _p(RR))
    D = D.T
    RR = RR.T
    iu = np.triu_indices(n)
    den = RR[iu]
    num = np.abs(D[iu])
    mask = den > 0
    return float((num[mask] / den[mask]).max()) if mask.any() else 0.0


# ------------------------------------------------ tridiagonal A (NEXT-N3) ---
def _vec(v):
    v = np.ascontiguousarray(v, dtype=np.float64)
    return v if v.size else np.zeros(1)


def gram_tridiag(d, e, Z, m):
    """G = Z^T (T Z), T = tridiag(e, d, e); storage (n, n)."""
    Z, ldz = _cm(Z, m)
    n = Z.shape[0]
    G = np.empty((n, n))
    d, e = _vec(d), _vec(e)
    _load().orc_gram_tridiag(m, n, _p(d), _p(e), _p(Z), ldz, _p(G), n)
    return G


def _variant_tridiag(fn, d, e, Z, m):
    Z, ldz = _cm(Z, m)
    n = Z.shape[0]
    Q = np.zeros((n, m))
    R = np.zeros((n, n))
    d, e = _vec(d), _vec(e)
    info = getattr(_load(), fn)(m, n, _p(d), _p(e), _p(Z), ldz, _p(Q), _p(R))
    return Q, R, info


def normal_tridiag(d, e, Z, m):
    return _variant_tridiag("orc_normal_tridiag", d, e, Z, m)


def normal2_tridiag(d, e, Z, m):
    return _variant_tridiag("orc_normal2_tridiag", d, e, Z, m)


def prequr_tridiag(d, e, Z, m):
    return _variant_tridiag("orc_prequr_tridiag", d, e, Z, m)


VARIANTS_TRIDIAG = {"normal": normal_tridiag, "normal2": normal2_tridiag, "prequr": prequr_tridiag}


def orth_error_tridiag(d, e, Q, m) -> float:
    """||Q^T T Q - I||_2, check formed in double-double."""
    Q, ldq = _cm(Q, m)
    n = Q.shape[0]
    E = np.empty((n, n))
    d, e = _vec(d), _vec(e)
    _load().orc_dd_orth_tridiag(m, n, _p(d), _p(e), _p(Q), ldq, _p(E))
    return float(np.linalg.norm(E.T, 2))


def densify_tridiag(d, e):
    """Dense column-major storage (m, m) of tridiag(e, d, e) (for pins and small checks)."""
    m = len(d)
    A = np.diag(np.asarray(d, dtype=np.float64))
    if m > 1:
        A += np.diag(np.asarray(e, dtype=np.float64), 1) + np.diag(np.asarray(e, dtype=np.float64), -1)
    return to_cm(A)
