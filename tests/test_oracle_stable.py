"""Pins for the stable pre-step (NEXT-N1, reading R21): shifted CholeskyQR3 and PRE-CHOLQR on it.

* scqr3 is a backward-stable Euclidean QR for kappa(Z) up to ~1e14: ||Y^T Y - I|| = O(n u) and
  ||Z - Y S|| / ||Z|| = O(u), and S equals the Householder R (LAPACK, positive diagonal) to
  O(u kappa(Z)) -- the properties Theorem 3 assumes of the pre-step;
* where the Euclidean Cholesky-QR pre-step (reading R2) breaks down (kappa(Z) = 1e10, 1e12),
  prequr_stable succeeds with Theorem 3's O(u ||A|| ||Q||^2) orthogonality;
* A = I reduces to Euclidean QR.
"""
import numpy as np
import pytest

import gen
import oracle
from oracle import U, from_cm, to_cm


@pytest.mark.parametrize("kz", [1e2, 1e8, 1e12, 1e14])
def test_scqr3_is_stable_euclidean_qr(kz):
    m, n = 400, 12
    p = gen.problem(m, n, 1.0, kz, 51, with_A=False)
    Y, S, info = oracle.scqr3(p.Z, m)
    assert info == 0
    Yd, Sd, Zd = from_cm(Y, m), from_cm(S, n), from_cm(p.Z, m)
    assert np.linalg.norm(Yd.T @ Yd - np.eye(n), 2) <= 10 * n * U
    assert np.linalg.norm(Zd - Yd @ Sd, 2) / np.linalg.norm(Zd, 2) <= 10 * n * U
    _, Rh = np.linalg.qr(Zd)
    Rh = Rh * np.sign(np.diag(Rh))[:, None]
    assert np.linalg.norm(Sd - Rh) / np.linalg.norm(Rh) <= 10 * n * U * kz


@pytest.mark.parametrize("kz", [1e10, 1e12])
def test_prequr_stable_where_cholqr_prestep_breaks_down(kz):
    m, n, ka = 400, 12, 1e6
    p = gen.problem(m, n, ka, kz, 52)
    _, _, info_plain = oracle.prequr(p.A, p.Z, m)
    assert 1 <= info_plain <= n                      # the Euclidean Cholesky-QR pre-step fails
    Q, R, info = oracle.prequr_stable(p.A, p.Z, m)
    assert info == 0
    E = oracle.orth_error(p.A, Q, m)
    scale = U * float(np.max(p.d)) * np.linalg.norm(from_cm(Q, m), 2) ** 2
    assert E <= 10 * n * scale
    assert oracle.componentwise_ratio(p.Z, Q, R, m) <= 100 * U * n


def test_prequr_stable_identity_is_euclidean_qr():
    m, n = 300, 9
    p = gen.problem(m, n, 1.0, 1e11, 53, with_A=False)
    Q, R, info = oracle.prequr_stable(to_cm(np.eye(m)), p.Z, m)
    assert info == 0
    _, Rh = np.linalg.qr(from_cm(p.Z, m))
    Rh = Rh * np.sign(np.diag(Rh))[:, None]
    assert np.linalg.norm(from_cm(R, n) - Rh) / np.linalg.norm(Rh) <= 10 * n * U * 1e11
