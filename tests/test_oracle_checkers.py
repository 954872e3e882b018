"""Pins for the oracle's double-double CHECKERS (orc_dd_gram, orc_dd_resid, orc_dd_chol_resid,
orc_dd_orth, orc_dd_orth_cols, orc_dd_orth_tridiag) and the Python reductions built on them
(componentwise_ratio, repr_error, chol_backward_ratio, orth_error).

The checkers compute the quantities the paper's error statements are about:
  G = Z^T A Z and M = |Z|^T |A| |Z|           eq.mult1-2
  G - R^T R and |R|^T |R|                      eq:normal:chol, PAPER.md:195-196
  Z - QR and |Q| |R|                           PAPER.md:197-198, Theorem 2
  Q^T A Q - I                                  PAPER.md:760 (orthogonality error)
  ||Z - QR|| / ||Z||                           PAPER.md:761 (representativity error)
They set the tolerances of the GPU gates, so each is pinned here against EXACT rational
arithmetic (Python fractions on the FP64 inputs, m <= 8) on inputs whose exact result is known
and NONZERO, and chosen so that plain FP64 evaluation of the same quantity would miss the pin:
the exact value is of the size of the FP64 rounding error of forming it (cancellation), which
only a correct double-double accumulation resolves.  A wrong checker (dropped low-order term,
missing fabs, off-by-one range, missing -I, transposed operand) fails one of these pins
(tests/oracle_mutation_check.py applies those mutations).

Bounds used.  A double-double accumulation of N products, rounded once at the end, satisfies
|x_dd - x| <= u |x| + c N u^2 S, with S the sum of the absolute values of the terms (each
TwoProd is exact; each dd addition loses O(u^2) relative to its running magnitude).  We use
c = 8.  A sum of N nonnegative FP64 terms satisfies |s - x| <= gamma_N x.
"""
from fractions import Fraction

import numpy as np
import pytest

import oracle
from oracle import U, from_cm, gamma, to_cm

F = Fraction


def fr(M):
    M = np.atleast_2d(np.asarray(M, dtype=np.float64))
    return [[F(float(v)) for v in row] for row in M]


def mm(X, Y):
    return [[sum((X[i][t] * Y[t][j] for t in range(len(Y))), F(0)) for j in range(len(Y[0]))]
            for i in range(len(X))]


def tr(X):
    return [list(r) for r in zip(*X)]


def absf(X):
    return [[abs(v) for v in row] for row in X]


def to_np(X):
    return np.array([[float(v) for v in row] for row in X])


def err(x_np, X_exact):
    """|x - X| entrywise, computed exactly then rounded."""
    return np.array([[float(abs(F(float(x_np[i, j])) - X_exact[i][j])) for j in range(x_np.shape[1])]
                     for i in range(x_np.shape[0])])


def dd_bound(X_exact, S_np, nterms):
    return U * np.abs(to_np(X_exact)) + 8 * nterms * U * U * S_np + 1e-300


def cancelling_problem(seed, m=8, n=3, symmetric=False):
    """A (m x m, nonsymmetric unless asked) and Z (m x n) with Z^T A Z's off-diagonal entries
    cancelled down to rounding level: column 2 of Z is made A-orthogonal to column 0 (and column
    1 to column 0 from the other side) in FP64, so the exact entries are O(u)|Z|^T|A||Z|."""
    rng = np.random.default_rng(seed)
    A = rng.standard_normal((m, m)) + m * np.eye(m)
    if symmetric:
        A = 0.5 * (A + A.T)
    Z = rng.standard_normal((m, n))
    z0 = Z[:, 0]
    v = Z[:, 2]
    # z0^T A z2 ~ 0: subtract along e_0 scaled by (z0^T A e_0)
    Z[0, 2] = v[0] - (z0 @ (A @ v)) / (z0 @ A[:, 0])
    v = Z[:, 1]
    Z[0, 1] = v[0] - ((A @ z0) @ v) / ((A @ z0)[0])   # (A z0)^T z1 ~ 0, i.e. z1^T A z0 ~ 0
    return A, Z


# ---------------------------------------------------------------- orc_dd_gram ----
@pytest.mark.parametrize("seed", [1, 2, 3])
def test_dd_gram_exact(seed):
    m, n = 8, 3
    A, Z = cancelling_problem(seed, m, n)
    G, M = oracle.dd_gram(to_cm(A), to_cm(Z), m)
    Af, Zf = fr(A), fr(Z)
    Ge = mm(tr(Zf), mm(Af, Zf))
    Me = mm(tr(absf(Zf)), mm(absf(Af), absf(Zf)))
    Me_np = to_np(Me)
    # the pin is sharp: the cancelled entries are below the FP64 evaluation error
    assert abs(float(Ge[0][2])) < 1e-12 * Me_np[0, 2] and abs(float(Ge[1][0])) < 1e-12 * Me_np[1, 0]
    assert abs(float(Ge[0][2])) > 0 and abs(float(Ge[1][0])) > 0            # known, nonzero
    plain = Z.T @ (A @ Z)
    assert np.any(err(plain, Ge) > dd_bound(Ge, Me_np, 2 * m)), "input does not discriminate"
    assert np.all(err(G, Ge) <= dd_bound(Ge, Me_np, 2 * m)), err(G, Ge) / dd_bound(Ge, Me_np, 2 * m)
    # M: nonnegative sums, relative gamma_{2m}
    assert np.all(err(M, Me) <= gamma(2 * m) * Me_np)
    # nonsymmetric A: G is not symmetric, and the checker keeps the orientation Z^T A Z
    assert abs(float(Ge[0][1] - Ge[1][0])) > 1e-3


# ---------------------------------------------------------------- orc_dd_resid ---
def _resid_case(seed, m=8, n=4, perturb=0.0):
    rng = np.random.default_rng(seed)
    A = rng.standard_normal((m, m))
    A = A @ A.T + m * np.eye(m)
    Z = rng.standard_normal((m, n))
    Q, R, info = oracle.normal(to_cm(A), to_cm(Z), m)
    assert info == 0
    Qd, Rd = from_cm(Q, m), from_cm(R, n)
    if perturb:
        Qd = Qd.copy()
        Qd[3, 1] += perturb
    return Z, Qd, Rd


@pytest.mark.parametrize("seed,perturb", [(4, 0.0), (5, 0.0), (6, 1e-9)])
def test_dd_resid_exact(seed, perturb):
    m, n = 8, 4
    Z, Q, R = _resid_case(seed, m, n, perturb)
    D, QRabs = oracle.dd_resid(to_cm(Z), to_cm(Q), to_cm(R), m)
    Zf, Qf, Rf = fr(Z), fr(Q), fr(R)
    QR = mm(Qf, Rf)
    De = [[Zf[i][j] - QR[i][j] for j in range(n)] for i in range(m)]
    Ae = mm(absf(Qf), absf(Rf))
    Ae_np = to_np(Ae)
    assert any(De[i][j] != 0 for i in range(m) for j in range(n))      # known, nonzero residual
    plain = Z - Q @ R
    if not perturb:
        # the residual of a computed factorization is O(u)|Q||R|: FP64 evaluation cannot resolve it
        assert np.any(err(plain, De) > dd_bound(De, Ae_np, n + 1))
    assert np.all(err(D, De) <= dd_bound(De, Ae_np, n + 1)), (err(D, De) / dd_bound(De, Ae_np, n + 1)).max()
    assert np.all(err(QRabs, Ae) <= gamma(n) * Ae_np)
    if perturb:                                     # the perturbed entry shows up where it must
        assert abs(D[3, 1] + perturb * R[1, 1]) <= 1e-6 * perturb * R[1, 1]


def test_componentwise_and_repr_error_exact():
    """rho = max |Z - QR|_ij / (|Q||R|)_ij and ||Z - QR||_2 / ||Z||_2 against
    exact residuals."""
    m, n = 8, 4
    for seed, pert in ((7, 0.0), (8, 3e-10)):
        Z, Q, R = _resid_case(seed, m, n, pert)
        Zf, Qf, Rf = fr(Z), fr(Q), fr(R)
        QR = mm(Qf, Rf)
        De = to_np([[Zf[i][j] - QR[i][j] for j in range(n)] for i in range(m)])
        Ae = to_np(mm(absf(Qf), absf(Rf)))
        mask = Ae > U * np.abs(Z).max()
        rho_exact = (np.abs(De)[mask] / Ae[mask]).max()
        rho = oracle.componentwise_ratio(to_cm(Z), to_cm(Q), to_cm(R), m)
        assert rho_exact > 0
        assert abs(rho - rho_exact) <= 1e-6 * rho_exact, (rho, rho_exact)
        rep = oracle.repr_error(to_cm(Z), to_cm(Q), to_cm(R), m)
        rep_exact = np.linalg.norm(De, 2) / np.linalg.norm(Z, 2)
        assert abs(rep - rep_exact) <= 1e-6 * rep_exact, (rep, rep_exact)


# ------------------------------------------------------------ orc_dd_chol_resid ---
@pytest.mark.parametrize("seed", [9, 10])
def test_dd_chol_resid_exact(seed):
    n = 6
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((n + 2, n))
    G = X.T @ X
    R, info = oracle.potrf(to_cm(G))
    assert info == 0
    Rd = from_cm(R, n)
    Gf, Rf = fr(G), fr(Rd)
    RtR = mm(tr(Rf), Rf)
    De = [[Gf[i][j] - RtR[i][j] for j in range(n)] for i in range(n)]
    Ae = mm(tr(absf(Rf)), absf(Rf))
    Ae_np = to_np(Ae)
    iu = np.triu_indices(n)
    # raw checker outputs (upper triangle is what it defines)
    Gc = to_cm(G)
    D = np.empty((n, n))
    RR = np.empty((n, n))
    lib = oracle._load()
    lib.orc_dd_chol_resid(n, oracle._p(Gc), n, oracle._p(np.ascontiguousarray(R)), n, oracle._p(D), oracle._p(RR))
    D, RR = D.T, RR.T
    e = err(D, De)[iu]
    b = dd_bound(De, Ae_np, n + 1)[iu]
    assert any(De[i][j] != 0 for i, j in zip(*iu))
    assert np.any(err(G - Rd.T @ Rd, De)[iu] > b), "input does not discriminate"
    assert np.all(e <= b), (e / b).max()
    assert np.all(err(RR, Ae)[iu] <= gamma(n) * Ae_np[iu])
    ratio = oracle.chol_backward_ratio(G, R)
    mask = Ae_np[iu] > 0
    ratio_exact = (np.abs(to_np(De))[iu][mask] / Ae_np[iu][mask]).max()
    assert ratio_exact > 0 and abs(ratio - ratio_exact) <= 1e-6 * ratio_exact


# ---------------------------------------------------------------- orc_dd_orth ----
def _orth_exact(A, Q):
    Af, Qf = fr(A), fr(Q)
    E = mm(tr(Qf), mm(Af, Qf))
    for i in range(len(E)):
        E[i][i] -= 1
    S = to_np(mm(tr(absf(Qf)), mm(absf(Af), absf(Qf))))
    return E, S


@pytest.mark.parametrize("seed,nonsym", [(11, False), (12, True)])
def test_dd_orth_exact(seed, nonsym):
    """E = Q^T A Q - I for a computed A-orthonormal Q (E = O(u), FP64 evaluation cannot resolve
    it) and for a Q that is not A-orthonormal; nonsymmetric A catches a transposed operand."""
    m, n = 8, 4
    rng = np.random.default_rng(seed)
    A = rng.standard_normal((m, m))
    A = A @ A.T + m * np.eye(m)
    Z = rng.standard_normal((m, n))
    Q, _, info = oracle.normal(to_cm(A), to_cm(Z), m)
    assert info == 0
    Qd = from_cm(Q, m)
    if nonsym:
        A = A + 0.25 * np.triu(rng.standard_normal((m, m)), 1)
    for Qx in (Qd, Qd + 1e-3 * rng.standard_normal((m, n))):
        Ee, S = _orth_exact(A, Qx)
        E = oracle.dd_orth_matrix(to_cm(A), to_cm(Qx), m)
        b = dd_bound(Ee, S, 2 * m)
        assert np.all(err(E, Ee) <= b), (err(E, Ee) / b).max()
        assert any(v != 0 for row in Ee for v in row)
        En = to_np(Ee)
        assert abs(oracle.orth_error(to_cm(A), to_cm(Qx), m) - np.linalg.norm(En, 2)) <= 1e-6 * np.linalg.norm(En, 2)
        cols = [0, 2, 3]
        Es = oracle.dd_orth_cols(to_cm(A), to_cm(Qx), m, cols)
        assert np.all(err(Es, [[Ee[i][j] for j in cols] for i in cols]) <= b[np.ix_(cols, cols)])
    if not nonsym:
        plain = Qd.T @ A @ Qd - np.eye(n)
        Ee, S = _orth_exact(A, Qd)
        assert np.any(err(plain, Ee) > dd_bound(Ee, S, 2 * m)), "input does not discriminate"


def test_dd_orth_tridiag_exact():
    m, n = 8, 3
    rng = np.random.default_rng(13)
    d = 4.0 + rng.random(m)
    e = rng.standard_normal(m - 1)          # non-constant: an index slip in the stencil fails
    T = np.diag(d) + np.diag(e, 1) + np.diag(e, -1)
    Z = rng.standard_normal((m, n))
    Q, _, info = oracle.normal(to_cm(T), to_cm(Z), m)
    assert info == 0
    Qd = from_cm(Q, m)
    for Qx in (Qd, Qd + 1e-4 * rng.standard_normal((m, n))):
        Ee, S = _orth_exact(T, Qx)
        Ec = np.empty((n, n))
        oracle._load().orc_dd_orth_tridiag(m, n, oracle._p(d), oracle._p(e), oracle._p(to_cm(Qx)), m, oracle._p(Ec))
        b = dd_bound(Ee, S, 2 * 3)
        assert np.all(err(Ec.T, Ee) <= b), (err(Ec.T, Ee) / b).max()


def test_dd_orth_euclid_exact():
    """Y^T Y - I for a Householder Y (E = O(u)) and a perturbed one, against exact arithmetic."""
    m, n = 8, 4
    rng = np.random.default_rng(14)
    Y, _ = oracle.hhqr(to_cm(rng.standard_normal((m, n))), m)
    Yd = from_cm(Y, m)
    for Yx in (Yd, Yd + 1e-5 * rng.standard_normal((m, n))):
        Ee, S = _orth_exact(np.eye(m), Yx)
        E = oracle.dd_orth_euclid_matrix(to_cm(Yx), m)
        b = dd_bound(Ee, S, m)
        assert any(v != 0 for row in Ee for v in row)
        assert np.all(err(E, Ee) <= b), (err(E, Ee) / b).max()
    Ee, S = _orth_exact(np.eye(m), Yd)
    assert np.any(err(Yd.T @ Yd - np.eye(n), Ee) > dd_bound(Ee, S, m)), "input does not discriminate"
