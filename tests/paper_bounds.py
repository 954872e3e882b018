"""Evaluators of the paper's error bounds on computed factors (test infrastructure; numpy norms
as library primitives).  Constants c = 1 (the paper omits them when plotting).

Theorem 2 (CHOLQR):
  normwise representativity   ||Z - QR||_2 <= n u ||Q||_2 ||R||_2                   (eq.repres)
  componentwise               |Z - QR| <= n u |Q||R|   ->  ||Z - QR||_2 <= n u || |Q||R| ||_2
  orthogonality               ||Q^T A Q - I||_2 <= m n u ||R^-1|| ||Z|| (||R^-1|| ||A Z|| + ||Q|| ||A||)  (eq.orth1)
Theorem 3 (PRE-CHOLQR):
  ||Z - QR||_2 <= m n^2 u ||Q|| ||U|| ||S||  (we use ||Q|| ||R|| <= ||Q|| ||U|| ||S||: a stronger check)
  ||Q^T A Q - I||_2 <= m n^2 u ||Q||^2 ||A||
All bounds are returned relative where the paper plots them relative (representativity / ||Z||).
"""
import numpy as np

U = 2.0 ** -53


def _n2(X):
    return float(np.linalg.norm(X, 2))


def thm2(A, Z, Q, R, normA):
    m, n = Z.shape
    smin = np.linalg.svd(R, compute_uv=False)[-1]
    nz = _n2(Z)
    rinv = 1.0 / smin if smin > 0 else np.inf
    return dict(
        repr_norm=n * U * _n2(Q) * _n2(R) / nz,
        repr_comp=n * U * _n2(np.abs(Q) @ np.abs(R)) / nz,
        orth1=m * n * U * rinv * nz * (rinv * _n2(A @ Z) + _n2(Q) * normA),
    )


def thm3(m, n, Q, R, Z, normA):
    return dict(
        repr_norm=m * n * n * U * _n2(Q) * _n2(R) / _n2(Z),
        orth=m * n * n * U * _n2(Q) ** 2 * normA,
    )


def slope(xs, ys):
    """Least-squares slope of log10 y against log10 x."""
    return float(np.polyfit(np.log10(xs), np.log10(ys), 1)[0])
