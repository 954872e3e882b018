"""Seeded synthetic input generator (shared by the CUDA path's tests/bench and the oracle).

Input generation only: no method arithmetic lives here (see ``oqr_gen.c`` header for the
recipe and its citations: SURVEY.md s8(d), BASELINE.json configs).

Matrices are column-major.  A column-major ``rows x cols`` matrix with leading dimension
``ld`` is held in a C-contiguous numpy array of shape ``(cols, ld)`` (``arr[j, i]`` is
element ``(i, j)``), which is also how the C ABI and the oracle take it.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboqr_gen.so")

REFLECT, BOTTOM, TOP, SPLIT, RANDOM, AORTH = 0, 1, 2, 3, 4, 5
UCASES = {"reflect": REFLECT, "bottom": BOTTOM, "top": TOP, "split": SPLIT, "random": RANDOM, "aorth": AORTH}
# the paper's case numbers
PAPER_CASES = {1: "bottom", 2: "top", 3: "split", 4: "random", 5: "aorth"}

SEED_BASE = 0x14015171

# BASELINE.json configs[0..4] (m, n, kappa_A, kappa_Z); seed_k = 0x14015171 + k.
CONFIGS = {
    0: dict(m=200, n=10, kappa_a=1e2, kappa_z=1e2),
    1: dict(m=4000, n=50, kappa_a=1e4, kappa_z=1e3),
    2: dict(m=20000, n=100, kappa_a=1e2, kappa_z=1e2),
    3: dict(m=40000, n=200, kappa_a=1e3, kappa_z=1e2),
    4: dict(m=10000, n=100, kappa_a=1e8, kappa_z=1e6),
}


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "oqr_gen.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        cmd = f"gcc -O2 -ffp-contract=off -fno-fast-math -fopenmp -fPIC -shared -Wall -o {_LIB_PATH} {src} -lm"
        if os.system(cmd) != 0:
            raise RuntimeError("failed to build gen/liboqr_gen.so: " + cmd)
    return _LIB_PATH


_lib = None


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB_PATH)
        P = ctypes.c_void_p
        lib.oqr_gen_problem.restype = ctypes.c_int
        lib.oqr_gen_problem.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_double, ctypes.c_double,
                                        ctypes.c_uint64, ctypes.c_int, P, ctypes.c_int64, P, ctypes.c_int64,
                                        P, P, P, P, P, P, P, P, P]
        lib.oqr_gen_A_rows.restype = ctypes.c_int
        lib.oqr_gen_A_rows.argtypes = [ctypes.c_int64, ctypes.c_double, ctypes.c_uint64, ctypes.c_int64,
                                       ctypes.c_int64, P, ctypes.c_int64]
        lib.oqr_gen_problem_haar.restype = ctypes.c_int
        lib.oqr_gen_problem_haar.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_double, ctypes.c_double,
                                             ctypes.c_uint64, ctypes.c_int, P, ctypes.c_int64, P, ctypes.c_int64,
                                             P, P, P, P, P]
        lib.oqr_gen_normal.restype = ctypes.c_double
        lib.oqr_gen_normal.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64]
        _lib = lib
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


@dataclass
class Problem:
    """A generated instance plus the ground-truth factors of its construction."""
    m: int
    n: int
    kappa_a: float
    kappa_z: float
    seed: int
    ucase: str
    A: np.ndarray | None          # (m, lda) C-order == column-major m x m
    Z: np.ndarray                 # (n, ldz) C-order == column-major m x n
    Yv: np.ndarray                # (4, m): V = I - Yv^T-cols T Yv^T
    Tv: np.ndarray                # (4, 4) column-major upper triangular (Tv[c, a] = T[a, c])
    d: np.ndarray                 # (m,) eigenvalues of A, descending
    s: np.ndarray                 # (n,) singular values of Z, descending
    Yu: np.ndarray
    Tu: np.ndarray
    Yw: np.ndarray
    Tw: np.ndarray
    cols: np.ndarray              # (n,) V-columns used as left singular vectors, or -1
    extra: dict = field(default_factory=dict)

    @property
    def lda(self) -> int:
        return self.A.shape[1] if self.A is not None else self.m

    @property
    def ldz(self) -> int:
        return self.Z.shape[1]


def problem(m: int, n: int, kappa_a: float, kappa_z: float, seed: int, ucase: str = "reflect",
            with_A: bool = True, lda: int | None = None, ldz: int | None = None,
            A_out: np.ndarray | None = None, Z_out: np.ndarray | None = None) -> Problem:
    """Generate (A, Z).  ``A_out``/``Z_out`` may be preallocated (e.g. pinned) float64
    C-contiguous arrays of shape (m, lda) / (n, ldz)."""
    lib = _load()
    lda = m if lda is None else lda
    ldz = m if ldz is None else ldz
    A = None
    if with_A:
        A = A_out if A_out is not None else np.empty((m, lda), dtype=np.float64)
        assert A.shape == (m, lda) and A.dtype == np.float64 and A.flags.c_contiguous
        lda = A.shape[1]
    Z = Z_out if Z_out is not None else np.empty((n, ldz), dtype=np.float64)
    assert Z.shape[0] == n and Z.dtype == np.float64 and Z.flags.c_contiguous
    ldz = Z.shape[1]
    # padding rows (lda/ldz > m) are never part of the matrix: poison them with NaN so that a
    # kernel reading past row m shows up as a NaN result instead of adding silent zeros
    if lda > m and A is not None and A_out is None:
        A[:, m:] = np.nan
    if ldz > m and Z_out is None:
        Z[:, m:] = np.nan
    Yv = np.empty((4, m)); Tv = np.empty((4, 4)); d = np.empty(m); s = np.empty(n)
    Yu = np.zeros((4, m)); Tu = np.empty((4, 4)); Yw = np.empty((4, n)); Tw = np.empty((4, 4))
    cols = np.empty(n, dtype=np.int64)
    rc = lib.oqr_gen_problem(m, n, float(kappa_a), float(kappa_z), seed, UCASES[ucase],
                             _ptr(A), lda, _ptr(Z), ldz, _ptr(Yv), _ptr(Tv), _ptr(d), _ptr(s),
                             _ptr(Yu), _ptr(Tu), _ptr(Yw), _ptr(Tw), _ptr(cols))
    if rc != 0:
        raise ValueError(f"oqr_gen_problem rejected arguments (m={m}, n={n}, ucase={ucase})")
    return Problem(m, n, kappa_a, kappa_z, seed, ucase, A, Z, Yv, Tv, d, s, Yu, Tu, Yw, Tw, cols)


@dataclass
class HaarProblem:
    """The paper's s7 construction with dense random orthogonal V, W (and U for case 4)."""
    m: int
    n: int
    kappa_a: float
    kappa_z: float
    seed: int
    ucase: str
    A: np.ndarray | None          # (m, lda) C-order == column-major m x m
    Z: np.ndarray                 # (n, ldz)
    V: np.ndarray                 # dense m x m eigenvectors of A (row-major numpy matrix)
    d: np.ndarray                 # (m,) eigenvalues, descending
    s: np.ndarray                 # (n,) singular values of Z, descending (case 5: d_J^{-1/2})
    W: np.ndarray                 # dense n x n right singular vectors
    cols: np.ndarray              # (n,) V-columns used as left singular vectors, or -1 (case 4)


def problem_haar(m: int, n: int, kappa_a: float, kappa_z: float, seed: int, ucase: str = "random",
                 with_A: bool = True, lda: int | None = None, ldz: int | None = None) -> HaarProblem:
    """A = V diag(d) V^T with V = orth(randn(m)); Z = U diag(s) W^T with W =
    orth(randn(n)) and U the case's columns of V (cases 1, 2, 3, 5) or orth(randn(m, n)) (case 4,
    ucase="random").  m <= 4096 (dense O(m^3) construction).  Padding rows are NaN."""
    lib = _load()
    lda = m if lda is None else lda
    ldz = m if ldz is None else ldz
    A = np.full((m, lda), np.nan) if with_A else None
    Z = np.full((n, ldz), np.nan)
    V = np.empty((m, m)); d = np.empty(m); s = np.empty(n); W = np.empty((n, n))
    cols = np.empty(n, dtype=np.int64)
    rc = lib.oqr_gen_problem_haar(m, n, float(kappa_a), float(kappa_z), seed, UCASES[ucase], _ptr(A), lda,
                                  _ptr(Z), ldz, _ptr(V), _ptr(d), _ptr(s), _ptr(W), _ptr(cols))
    if rc != 0:
        raise ValueError(f"oqr_gen_problem_haar rejected arguments (m={m}, n={n}, ucase={ucase})")
    # V, W come back column-major: V[k] is column k -> transpose to dense matrices
    return HaarProblem(m, n, kappa_a, kappa_z, seed, ucase, A, Z, V.T.copy(), d, s, W.T.copy(), cols)


def A_rows(m: int, kappa_a: float, seed: int, r0: int, r1: int, lda: int | None = None,
           out: np.ndarray | None = None) -> np.ndarray:
    """Rows [r0, r1) of the A that ``problem(m, ..., kappa_a, ..., seed)`` generates (bitwise the
    same entries) as a column-major (r1-r0) x m block: C-contiguous array of shape (m, lda)."""
    lda = (r1 - r0) if lda is None else lda
    a = out if out is not None else np.empty((m, lda), dtype=np.float64)
    assert a.shape == (m, lda) and a.dtype == np.float64 and a.flags.c_contiguous
    rc = _load().oqr_gen_A_rows(m, float(kappa_a), seed, r0, r1, _ptr(a), lda)
    if rc != 0:
        raise ValueError(f"oqr_gen_A_rows rejected arguments (m={m}, rows=[{r0},{r1}))")
    return a


def config_A_rows(k: int, r0: int, r1: int, **kw) -> np.ndarray:
    c = CONFIGS[k]
    return A_rows(c["m"], c["kappa_a"], SEED_BASE + k, r0, r1, **kw)


# NEXT-N3 tridiagonal workload (A tridiagonal, m = 100000, n varied).
# The paper does not give the entries of its tridiagonal A; we use the shifted 1-D Laplacian
# T = tridiag(-1, 2 + c, -1) with c chosen so that kappa(T) is exactly kappa_A (R18).
TRIDIAG_CONFIGS = {
    "T": dict(m=100000, n=200, kappa_a=1e3, kappa_z=1e2),      # bench / full-size parity
    "t": dict(m=2000, n=30, kappa_a=1e3, kappa_z=1e2),         # small parity case
}


def tridiag(m: int, kappa_a: float):
    """(d, e): diagonal (m) and off-diagonal (m-1) of T = tridiag(-1, 2 + c, -1), whose eigenvalues
    are lambda_k = c + 2 - 2 cos(k pi / (m + 1)) with eigenvectors sqrt(2/(m+1)) sin(i k pi/(m+1));
    c = 2 cos(pi/(m+1)) (kappa+1)/(kappa-1) - 2 makes lambda_m / lambda_1 = kappa_A.
    Input generation only (closed form, no method arithmetic)."""
    C = np.cos(np.pi / (m + 1))
    c = 2.0 * C * (kappa_a + 1.0) / (kappa_a - 1.0) - 2.0 if kappa_a > 1.0 else 0.0
    d = np.full(m, 2.0 + c)
    e = np.full(max(m - 1, 0), -1.0)
    return d, e


def tridiag_eigen(m: int, kappa_a: float, ks):
    """Exact eigenvalues lambda_k and unit eigenvectors (m x len(ks)) of tridiag(m, kappa_a), k 1-based."""
    C = np.cos(np.pi / (m + 1))
    c = 2.0 * C * (kappa_a + 1.0) / (kappa_a - 1.0) - 2.0 if kappa_a > 1.0 else 0.0
    ks = np.asarray(ks, dtype=np.float64)
    lam = c + 2.0 - 2.0 * np.cos(ks * np.pi / (m + 1))
    i = np.arange(1, m + 1, dtype=np.float64)[:, None]
    V = np.sqrt(2.0 / (m + 1)) * np.sin(i * ks[None, :] * np.pi / (m + 1))
    return lam, V


def tridiag_config(key: str, **kw):
    """(d, e, Problem with Z only) for TRIDIAG_CONFIGS[key]; Z as in the dense configs (ucase reflect)."""
    c = TRIDIAG_CONFIGS[key]
    d, e = tridiag(c["m"], c["kappa_a"])
    p = problem(c["m"], c["n"], c["kappa_a"], c["kappa_z"], SEED_BASE + 0x7D, with_A=False, **kw)
    return d, e, p


def config(k: int, ucase: str = "reflect", **kw) -> Problem:
    c = CONFIGS[k]
    return problem(c["m"], c["n"], c["kappa_a"], c["kappa_z"], SEED_BASE + k, ucase=ucase, **kw)


def witness(**kw) -> Problem:
    """Config-4 breakdown witness: same (m, n, kappa_A, kappa_Z), paper case 3 alignment
    (PAPER.md:730-732)."""
    return config(4, ucase="split", **kw)


def normal(seed: int, stream: int, k: int) -> float:
    return _load().oqr_gen_normal(seed, stream, k)


def wy_matrix(Y: np.ndarray, T: np.ndarray) -> np.ndarray:
    """Explicit I - Y T Y^T (rows x rows) from the generator's WY factors
    (Y given as (4, len), T column-major (4,4)).  For small pins only."""
    Ym = Y.T  # len x 4
    Tm = T.T  # row-major T[a, b]
    return np.eye(Ym.shape[0]) - Ym @ Tm @ Ym.T


def apply_wy(Y: np.ndarray, T: np.ndarray, X: np.ndarray, transpose: bool = False) -> np.ndarray:
    """(I - Y T Y^T) X, or its transpose applied, for X (len x k) in O(len*k)."""
    Ym = Y.T
    Tm = T.T
    M = Tm.T if transpose else Tm
    return X - Ym @ (M @ (Ym.T @ X))
