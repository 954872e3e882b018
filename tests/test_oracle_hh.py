"""Pins for the Householder pre-step of PRE-CHOLQR (NEXT-N1, paper-faithful Algorithm 2):
orc_geqr2 / orc_org2r / orc_hhqr / orc_prequr_hh (oracle/oqr_oracle.c).

Algorithm 2 line 1 is ``[Y,S] = qr(Z)`` with "a stable Euclidean QR factorization (such as
Householder QR)".  Pinned against:
  * SPEC's worked examples (tests/golden/spec_examples.json);
  * exact hand-derived reflectors on 2-vectors (beta, tau, v of the dlarfg convention);
  * LAPACK's QR (numpy.linalg.qr) with the same positive-diagonal normalisation, to the
    first-order forward-error bound u kappa(Z);
  * the backward-stability properties Theorem 3 assumes of the pre-step:
    ||Y^T Y - I|| <= c m n u and ||Z - Y S|| <= c m n u ||Z|| up to kappa(Z) = 1e15, where the
    Cholesky-based pre-steps fail;
  * A = I: PRE-CHOLQR is the Euclidean QR;
  * Theorem 3's orthogonality O(u ||A|| ||Q||^2) at kappa(Z) = 1e15.
"""
import json
import os

import numpy as np
import pytest

import gen
import oracle
from oracle import U, from_cm, to_cm

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def hh(Zd):
    m, n = Zd.shape
    Y, S = oracle.hhqr(to_cm(Zd), m)
    return from_cm(Y, m), from_cm(S, n)


def test_spec_examples():
    for key in ("householder_identity_cols", "householder_pythagorean"):
        g = GOLDEN[key]
        Y, S = hh(np.array(g["Z"]))
        assert np.array_equal(S, np.array(g["S"])), (key, S)
        assert np.allclose(Y, np.array(g["Y"]), rtol=0, atol=2 * U), (key, Y)
    g = GOLDEN["householder_random_bound"]
    Zd = np.random.default_rng(20).standard_normal((g["m"], g["n"]))
    Y, S = hh(Zd)
    assert np.linalg.norm(Y.T @ Y - np.eye(g["n"]), 2) <= g["orth_max"]
    assert np.linalg.norm(Zd - Y @ S, 2) / np.linalg.norm(Zd, 2) <= g["resid_max"]


def test_reflector_by_hand():
    """x = [0; -2]: alpha = 0, ||x|| = 2, beta = -2 (alpha >= 0 takes -sign), tau = (beta - alpha) /
    beta = 1, v = [1; x2 / (alpha - beta)] = [1; -1]; Y = H e1 = e1 - tau v = [0; 1], R = -2, and
    the positive-diagonal normalisation gives S = 2, Y = [0; -1] -- all exact."""
    X, tau = oracle.geqr2(to_cm(np.array([[0.0], [-2.0]])), 2)
    assert tau[0] == 1.0 and X[0, 0] == -2.0 and X[0, 1] == -1.0
    Y, S = hh(np.array([[0.0], [-2.0]]))
    assert S[0, 0] == 2.0 and np.array_equal(Y[:, 0], np.array([0.0, -1.0]))
    # x = [3; 4]: beta = -5, tau = (-5 - 3) / -5 = 1.6, v2 = 4 / 8 = 0.5 (exact in binary)
    X, tau = oracle.geqr2(to_cm(np.array([[3.0], [4.0]])), 2)
    assert tau[0] == 1.6 and X[0, 0] == -5.0 and X[0, 1] == 0.5


def test_reflectors_are_orthogonal():
    """H_j = I - tau_j v_j v_j^T is orthogonal iff tau_j (1 + ||v_tail||^2) = 2 (tau != 0)."""
    Zd = np.random.default_rng(21).standard_normal((30, 6))
    X, tau = oracle.geqr2(to_cm(Zd), 30)
    Xd = from_cm(X, 30)
    for j in range(6):
        vt = Xd[j + 1:, j]
        assert abs(tau[j] * (1.0 + vt @ vt) - 2.0) <= 8 * 30 * U


def test_zero_tail_column_is_left_alone():
    """A column already zero below the diagonal gets tau = 0 (H = I); a negative diagonal entry
    is then fixed by the sign normalisation alone."""
    Zd = np.array([[-3.0, 1.0], [0.0, 2.0], [0.0, 0.0]])
    X, tau = oracle.geqr2(to_cm(Zd), 3)
    assert tau[0] == 0.0 and tau[1] == 0.0
    Y, S = hh(Zd)
    assert np.array_equal(S, np.array([[3.0, -1.0], [0.0, 2.0]]))
    assert np.array_equal(Y, np.array([[-1.0, 0.0], [0.0, 1.0], [0.0, 0.0]]))


@pytest.mark.parametrize("kz", [1e2, 1e8, 1e12, 1e14, 1e15])
def test_backward_stable_to_1e15(kz):
    m, n = 400, 12
    p = gen.problem(m, n, 1.0, kz, 51, with_A=False)
    Y, S = oracle.hhqr(p.Z, m)
    Zd, Yd, Sd = from_cm(p.Z, m), from_cm(Y, m), from_cm(S, n)
    assert oracle.orth_error_euclid(Y, m) <= m * n * U
    D, _ = oracle.dd_resid(p.Z, Y, S, m)
    assert np.linalg.norm(D, 2) / np.linalg.norm(Zd, 2) <= m * n * U
    assert np.all(np.diag(Sd) > 0) and np.array_equal(Sd, np.triu(Sd))
    # LAPACK's Householder QR (positive-diagonal normalised): forward error of R <= c u kappa(Z)
    Qh, Rh = np.linalg.qr(Zd)
    sg = np.sign(np.diag(Rh))
    Rh = Rh * sg[:, None]
    assert np.linalg.norm(Sd - Rh) / np.linalg.norm(Rh) <= 10 * n * U * kz
    if kz <= 1e8:
        assert np.linalg.norm(Yd - Qh * sg) <= 10 * n * U * kz


def test_identity_A_is_euclidean_qr():
    m, n = 300, 9
    p = gen.problem(m, n, 1.0, 1e13, 53, with_A=False)
    Q, R, info = oracle.prequr_hh(to_cm(np.eye(m)), p.Z, m)
    assert info == 0
    Y, S = oracle.hhqr(p.Z, m)
    # CHOLQR of an orthonormal Y: U = I + O(u), Q = Y + O(u)
    assert np.linalg.norm(from_cm(Q, m) - from_cm(Y, m)) <= 10 * n * U * np.sqrt(n)
    assert np.linalg.norm(from_cm(R, n) - from_cm(S, n)) / np.linalg.norm(from_cm(S, n)) <= 10 * n * U


@pytest.mark.parametrize("kz", [1e10, 1e12, 1e14, 1e15])
def test_prequr_hh_theorem3(kz):
    """Where the Cholesky-based pre-steps break down (Euclidean CholQR from ~1e8, shifted
    CholeskyQR3 from ~1e13), the Householder pre-step gives Theorem 3's orthogonality
    ||Q^T A Q - I|| = O(u ||A|| ||Q||^2) and representativity O(u)."""
    m, n, ka = 400, 12, 1e6
    p = gen.problem(m, n, ka, kz, 52)
    Q, R, info = oracle.prequr_hh(p.A, p.Z, m)
    assert info == 0
    E = oracle.orth_error(p.A, Q, m)
    scale = U * float(np.max(p.d)) * np.linalg.norm(from_cm(Q, m), 2) ** 2
    assert E <= 10 * n * scale
    assert oracle.repr_error(p.Z, Q, R, m) <= 10 * n * U
    if kz >= 1e10:
        _, _, info_p = oracle.prequr(p.A, p.Z, m)
        assert info_p != 0        # the Euclidean Cholesky-QR pre-step is past its range here
