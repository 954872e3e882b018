"""Pins for the CPU oracle.  Each pin fixes the oracle against
something other than itself: values the paper/SPEC print (tests/golden/), exact rational
arithmetic, closed forms of the paper's s7 constructions, Theorem 1, LAPACK special cases,
and brute force with an explicit A^{1/2}.

These run on CPU (``-m "not gpu"``)."""
import json
import os
from fractions import Fraction

import numpy as np
import pytest

import gen
import oracle
from oracle import U, from_cm, gamma, to_cm

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def dense(a, rows):
    return from_cm(a, rows)


def svals(M):
    return np.linalg.svd(M, compute_uv=False)


# ------------------------------------------------------------------ P7 ----
def test_p7_cholesky_examples():
    for key in ("cholesky_2x2", "cholesky_identity3"):
        g = GOLDEN[key]
        R, info = oracle.potrf(to_cm(np.array(g["G"])))
        assert info == 0
        assert np.array_equal(dense(R, len(g["G"])), np.array(g["R"]))
    g = GOLDEN["cholesky_indefinite"]
    _, info = oracle.potrf(to_cm(np.array(g["G"])))
    assert info == g["info"]


def test_p7_cholesky_nan_breaks_down():
    G = np.eye(3)
    G[1, 1] = np.nan
    _, info = oracle.potrf(to_cm(G))
    assert info == 2


def test_p7_trsm_examples():
    g = GOLDEN["trsm_right"]
    B = np.array(g["B"])
    X = oracle.trsm(to_cm(B), to_cm(np.array(g["R"])), 1)
    assert np.allclose(dense(X, 1), np.array(g["X"]), rtol=0, atol=2 * U)
    Bi = np.random.default_rng(0).standard_normal((7, 4))
    Xi = oracle.trsm(to_cm(Bi), to_cm(np.eye(4)), 7)
    assert np.array_equal(dense(Xi, 7), Bi)


def test_p7_cholqr_pythagorean():
    g = GOLDEN["cholqr_pythagorean"]
    Q, R, info = oracle.normal(to_cm(np.array(g["A"])), to_cm(np.array(g["Z"])), 2)
    assert info == 0
    assert dense(R, 1)[0, 0] == 5.0
    assert np.array_equal(dense(Q, 2), np.array(g["Q"]))


# ------------------------------------------------------------------ P1 ----
def _householder_R(Z):
    Qh, Rh = np.linalg.qr(Z)
    sgn = np.sign(np.diag(Rh))
    return Qh * sgn, Rh * sgn[:, None]


@pytest.mark.parametrize("variant", ["normal", "normal2", "prequr"])
def test_p1_identity_reduces_to_euclidean_qr(variant):
    m, n, kz = 90, 8, 1e3
    p = gen.problem(m, n, 1.0, kz, 21, with_A=False)
    Z = dense(p.Z, m)
    Q, R, info = oracle.VARIANTS[variant](to_cm(np.eye(m)), p.Z, m)
    assert info == 0
    Qh, Rh = _householder_R(Z)
    Rd, Qd = dense(R, n), dense(Q, m)
    tol = 10 * n * U * kz ** 2
    assert np.linalg.norm(Rd - Rh) / np.linalg.norm(Rh) < tol
    assert np.linalg.norm(Qd - Qh) / np.linalg.norm(Qh) < tol
    orth = np.linalg.norm(Qd.T @ Qd - np.eye(n), 2)
    if variant == "normal":
        assert orth < tol
    else:  # a second pass restores orthogonality to O(u)
        assert orth < 100 * n * U


def test_p1_orthonormal_Z_gives_identity_R():
    m, n = 50, 5
    Zq, _ = np.linalg.qr(np.random.default_rng(1).standard_normal((m, n)))
    Q, R, info = oracle.normal(to_cm(np.eye(m)), to_cm(Zq), m)
    assert info == 0
    assert np.abs(dense(R, n) - np.eye(n)).max() < 1e-14
    assert np.abs(dense(Q, m) - Zq).max() < 1e-14


def test_p1_power_of_two_scaling_is_exact():
    """A = 4I: G = 4 Z^T Z and chol(4G) = 2 chol(G) exactly (power-of-two scaling commutes
    with rounding), so R(4I) = 2 R(I) and Q(4I) = Q(I)/2 bitwise."""
    m, n = 70, 6
    p = gen.problem(m, n, 1.0, 1e2, 3, with_A=False)
    Q1, R1, _ = oracle.normal(to_cm(np.eye(m)), p.Z, m)
    Q4, R4, _ = oracle.normal(to_cm(4.0 * np.eye(m)), p.Z, m)
    assert np.array_equal(R4, 2.0 * R1)
    assert np.array_equal(Q4, 0.5 * Q1)


# ------------------------------------------------------------------ P2 ----
def _sqrtA_times(p, X):
    """A^{1/2} X = V diag(sqrt d) V^T X from the generator's exact WY factors (O(mk))."""
    Y = gen.apply_wy(p.Yv, p.Tv, X, transpose=True)
    return gen.apply_wy(p.Yv, p.Tv, np.sqrt(p.d)[:, None] * Y)


@pytest.mark.parametrize("cfg", [0, 1])
def test_p2_theorem1_singular_values_of_R(cfg):
    """sigma_i(R) = sigma_i(A^{1/2} Z) (Theorem 1)."""
    p = gen.config(cfg)
    m, n = p.m, p.n
    Q, R, info = oracle.normal(p.A, p.Z, m)
    assert info == 0
    X = _sqrtA_times(p, dense(p.Z, m))
    sx = svals(X)
    sr = svals(dense(R, n))
    rel = np.abs(sr - sx) / sx
    gate = np.sqrt(m) * U * (sx[0] / sx) ** 2 * 10
    assert np.all(rel <= gate), (rel / gate).max()
    # ||Q||_2 = sigma_n(A^{1/2} Zhat)^{-1}
    Zhat, _ = np.linalg.qr(dense(p.Z, m))
    qn = np.linalg.norm(dense(Q, m), 2)
    ref = 1.0 / svals(_sqrtA_times(p, Zhat))[-1]
    kap = sx[0] / sx[-1]
    assert abs(qn / ref - 1.0) < 10 * np.sqrt(m) * U * kap ** 2


# ------------------------------------------------------------------ P3 ----
@pytest.mark.parametrize("cfg", [0, 1])
def test_p3_normal_equation(cfg):
    """Z^T A Z = R^T R: the oracle's G agrees with an independent
    LAPACK/BLAS product within eq.mult1-2, and R^T R reproduces G within the
    Cholesky backward error (eq:normal:chol)."""
    p = gen.config(cfg)
    m, n = p.m, p.n
    A, Z = dense(p.A, m), dense(p.Z, m)
    G = dense(oracle.gram(p.A, p.Z, m), n)
    Gb = Z.T @ (A @ Z)
    M = np.abs(Z).T @ np.abs(A) @ np.abs(Z)
    assert np.all(np.abs(G - Gb) <= 2 * gamma(2 * m) * M)
    R, info = oracle.potrf(to_cm(G))
    assert info == 0
    assert oracle.chol_backward_ratio(G, R) <= gamma(n + 1)
    Rd = dense(R, n)
    assert np.array_equal(Rd, np.triu(Rd)) and np.all(np.diag(Rd) > 0)


# ------------------------------------------------------------------ P4 ----
def _rational_matmul(X, Y):
    n, k = len(X), len(Y[0])
    return [[sum(X[i][t] * Y[t][j] for t in range(len(Y))) for j in range(k)] for i in range(n)]


def _frac(M):
    return [[Fraction(float(v)) for v in row] for row in M]


def test_p4_exact_rational_gram_nonsymmetric():
    """Exact G = Z^T A Z in rational arithmetic on the FP64 inputs; the oracle must satisfy
    |G - G_exact| <= gamma_{2m} |Z|^T |A| |Z| (eq.mult1-2).  A is NOT symmetric, so a transposed
    operand in the oracle fails this pin."""
    rng = np.random.default_rng(7)
    m, n = 8, 3
    A = rng.standard_normal((m, m))
    Z = rng.standard_normal((m, n))
    G = dense(oracle.gram(to_cm(A), to_cm(Z), m), n)
    Ge = _rational_matmul(_frac(Z.T), _rational_matmul(_frac(A), _frac(Z)))
    M = np.abs(Z).T @ np.abs(A) @ np.abs(Z)
    err = np.array([[abs(Fraction(float(G[i, j])) - Ge[i][j]) for j in range(n)] for i in range(n)], dtype=float)
    assert np.all(err <= gamma(2 * m) * M)
    # and a transposed A would be far outside it
    Gt = Z.T @ A.T @ Z
    assert np.abs(Gt - G).max() > 1e3 * (gamma(2 * m) * M).max()


def test_p4_exact_rational_cholesky_and_trsm():
    rng = np.random.default_rng(8)
    n, m = 5, 9
    X = rng.standard_normal((n + 3, n))
    G = X.T @ X
    R, info = oracle.potrf(to_cm(G))
    assert info == 0
    Rd = dense(R, n)
    Rf = _frac(Rd)
    RtR = _rational_matmul([list(r) for r in zip(*Rf)], Rf)
    for i in range(n):
        for j in range(i, n):
            bound = gamma(n + 1) * sum(abs(Rd[k, i]) * abs(Rd[k, j]) for k in range(n))
            assert abs(float(Fraction(float(G[i, j])) - RtR[i][j])) <= bound
    Z = rng.standard_normal((m, n))
    Q = dense(oracle.trsm(to_cm(Z), R, m), m)
    QR = _rational_matmul(_frac(Q), Rf)
    QRabs = np.abs(Q) @ np.abs(Rd)
    for i in range(m):
        for j in range(n):
            assert abs(float(Fraction(float(Z[i, j])) - QR[i][j])) <= gamma(n) * QRabs[i, j] + 1e-300


@pytest.mark.parametrize("variant", ["normal", "normal2", "prequr"])
@pytest.mark.parametrize("seed", [1, 2, 3])
def test_p4_brute_force_explicit_sqrtA(seed, variant):
    """R is the R factor of the Euclidean QR of A^{1/2} Z (Theorem 1 / SYEV-EQR,
    PAPER.md:504-511) and Q = C^{-1} Y for C = chol(A), [Y, R] = qr(C Z) (CHOL-EQR,
    PAPER.md:366-377 with the Q = C\\Y reading).  Explicit Haar V, m <= 64."""
    rng = np.random.default_rng(seed)
    m, n = 48, 6
    V, _ = np.linalg.qr(rng.standard_normal((m, m)))
    d = 10.0 ** (-np.linspace(0, 3, m))
    A = V @ np.diag(d) @ V.T
    A = 0.5 * (A + A.T)
    Z = rng.standard_normal((m, n)) @ np.diag(10.0 ** -np.linspace(0, 1, n))
    Q, R, info = oracle.VARIANTS[variant](to_cm(A), to_cm(Z), m)
    assert info == 0
    Rd, Qd = dense(R, n), dense(Q, m)
    X = V @ np.diag(np.sqrt(d)) @ V.T @ Z
    _, Rbf = _householder_R(X)
    kG = np.linalg.cond(X) ** 2
    assert np.linalg.norm(Rd - Rbf) / np.linalg.norm(Rbf) <= 10 * np.sqrt(m) * U * kG
    C = np.linalg.cholesky(A).T  # A = C^T C, C upper
    Yq, Rc = _householder_R(C @ Z)
    Qc = np.linalg.solve(C, Yq)
    assert np.linalg.norm(Qd - Qc) / np.linalg.norm(Qc) <= 10 * np.sqrt(m) * U * kG


# ------------------------------------------------------------------ P5 ----
def test_p5_closed_form_eigvec_columns_no_W():
    """Z = V_J diag(s) (no right rotation): G = diag(s^2 d_J) exactly in exact arithmetic,
    so R = diag(s sqrt(d_J)) and Q = V_J diag(d_J^{-1/2})."""
    m, n = 80, 10
    p = gen.problem(m, n, 1e6, 1e3, 31, ucase="split")
    V = gen.wy_matrix(p.Yv, p.Tv)
    J = p.cols
    Z = V[:, J] * p.s
    Q, R, info = oracle.normal(p.A, to_cm(Z), m)
    assert info == 0
    Rd, Qd = dense(R, n), dense(Q, m)
    Rexp = np.diag(p.s * np.sqrt(p.d[J]))
    kap = (Rexp.max() / Rexp[Rexp > 0].min())
    assert np.abs(Rd - Rexp).max() / Rexp.max() <= 10 * m * U * kap
    Qexp = V[:, J] / np.sqrt(p.d[J])
    assert np.linalg.norm(Qd - Qexp) / np.linalg.norm(Qexp) <= 10 * m * U * kap ** 2


@pytest.mark.parametrize("ucase", ["top", "bottom", "split"])
def test_p5_singular_values_closed_form(ucase):
    """Any W: sigma(R) = sort(s * sqrt(d_J)) (Theorem 1 + the s7 construction)."""
    m, n = 80, 10
    p = gen.problem(m, n, 1e4, 1e2, 41, ucase=ucase)
    _, R, info = oracle.normal(p.A, p.Z, m)
    assert info == 0
    sr = svals(dense(R, n))
    sx = np.sort(p.s * np.sqrt(p.d[p.cols]))[::-1]
    assert np.all(np.abs(sr - sx) / sx <= 10 * np.sqrt(m) * U * (sx[0] / sx) ** 2)


def test_p5_case5_aorthonormal():
    """Case 5: Z^T A Z = I so R = I and Q = Z."""
    m, n = 80, 10
    p = gen.problem(m, n, 1e8, 1.0, 51, ucase="aorth")
    Q, R, info = oracle.normal(p.A, p.Z, m)
    assert info == 0
    kap = p.s.max() / p.s.min()  # ||A|| ||Z||^2 = kappa(A) sets the size of the Gram error
    assert np.abs(dense(R, n) - np.eye(n)).max() <= 10 * m * U * kap ** 2
    assert np.linalg.norm(dense(Q, m) - dense(p.Z, m)) / np.linalg.norm(dense(p.Z, m)) <= 10 * m * U * kap ** 2


def test_p5_case2_and_case1_orth_constants():
    """||A|| ||Q||^2 = sigma_1(A)/sigma_n(A) for case 2 (golden 10^{54/79}) and
    = kappa(A) for cases 1 and 3."""
    g = GOLDEN["case2_orth_constant"]
    m, n, ka = g["m"], g["n"], g["kappa_a"]
    p = gen.problem(m, n, ka, 1e2, 61, ucase="top")
    Q, _, info = oracle.normal(p.A, p.Z, m)
    assert info == 0
    val = np.log10(np.linalg.norm(dense(Q, m), 2) ** 2 * p.d[0])
    assert abs(val - g["normA_normQ2_log10"]) < 1e-9
    for ucase in ("bottom", "split"):
        p = gen.problem(m, n, ka, 1e2, 62, ucase=ucase)
        Q, _, info = oracle.normal(p.A, p.Z, m)
        assert info == 0
        val = np.linalg.norm(dense(Q, m), 2) ** 2 * p.d[0]
        assert abs(val / ka - 1.0) < 1e-6


# ------------------------------------------------------------------ P6 ----
def test_p6_case2_cholqr_orth_proportional_to_kappaZ_squared():
    """CHOLQR loss of orthogonality is proportional to kappa(Z)^2 in case 2:
    slope of log E_orth vs log kappa(A) with kappa(Z) = kappa(A)^{1/2} is ~1."""
    m, n = 80, 10
    ks, es = [], []
    for e in range(2, 12):
        ka = 10.0 ** e
        p = gen.problem(m, n, ka, ka ** 0.5, 71, ucase="top")
        Q, R, info = oracle.normal(p.A, p.Z, m)
        assert info == 0
        err = oracle.orth_error(p.A, Q, m)
        ks.append(e)
        es.append(np.log10(err))
    slope = np.polyfit(ks, es, 1)[0]
    assert 0.8 <= slope <= 1.2, slope


@pytest.mark.parametrize("variant", ["normal2", "prequr"])
def test_p6_stable_variants_orth_bound(variant):
    """Thm 3: ||Q^T A Q - I|| <= c m n^2 u ||Q||^2 ||A||; observed O(u ||A|| ||Q||^2)
    for the stable algorithms.  Case 1 attains kappa(A)."""
    m, n = 80, 10
    for ucase, ka in (("top", 1e8), ("bottom", 1e6), ("split", 1e6)):
        p = gen.problem(m, n, ka, 1e3, 81, ucase=ucase)
        Q, R, info = oracle.VARIANTS[variant](p.A, p.Z, m)
        assert info == 0
        err = oracle.orth_error(p.A, Q, m)
        scale = U * p.d[0] * np.linalg.norm(dense(Q, m), 2) ** 2
        assert err <= 10 * n * scale, (ucase, err / scale)


@pytest.mark.parametrize("cfg", [0, 1])
def test_p6_componentwise_representativity(cfg):
    """|Z - QR| <= c n u |Q||R| (Theorem 2) with c = 1."""
    p = gen.config(cfg)
    Q, R, info = oracle.normal(p.A, p.Z, p.m)
    assert info == 0
    rho = oracle.componentwise_ratio(p.Z, Q, R, p.m)
    assert rho <= gamma(p.n + 1)


def test_p6_breakdown_witness_small():
    """Case 3 with kappa(A^{1/2} Z) >> u^{-1/2} breaks down;
    PRE-CHOLQR with a stable enough pre-step still succeeds."""
    m, n = 80, 10
    p = gen.problem(m, n, 1e15, 10 ** 7.5, 91, ucase="split")
    _, _, info = oracle.normal(p.A, p.Z, m)
    assert 1 <= info <= n
    _, _, info2 = oracle.normal2(p.A, p.Z, m)
    assert 1 <= info2 <= n
    p = gen.problem(m, n, 1e8, 1e6, 92, ucase="split")
    _, _, info = oracle.normal(p.A, p.Z, m)
    assert 1 <= info <= n
    Q, R, info3 = oracle.prequr(p.A, p.Z, m)
    assert info3 == 0


def test_trmm_and_variant_r_relation():
    """normal2: R = R2 R1 (upper x upper); the product is upper triangular."""
    rng = np.random.default_rng(3)
    n = 6
    R1 = np.triu(rng.standard_normal((n, n)))
    R2 = np.triu(rng.standard_normal((n, n)))
    R = dense(oracle.trmm(to_cm(R2), to_cm(R1)), n)
    assert np.allclose(R, R2 @ R1, rtol=0, atol=10 * n * U * (np.abs(R2) @ np.abs(R1)).max())
    assert np.array_equal(R, np.triu(R))


@pytest.mark.parametrize("variant", ["normal", "normal2", "prequr"])
@pytest.mark.parametrize("cfg", [0, 1])
def test_p6_variant_representativity(cfg, variant):
    """Z = QR to the Theorem 2/3 level for every variant: normwise
    ||Z - QR||/||Z|| = O(n u) and the R factors of all variants agree
    (uniqueness of the positive-diagonal factor)."""
    p = gen.config(cfg)
    m, n = p.m, p.n
    Q, R, info = oracle.VARIANTS[variant](p.A, p.Z, m)
    assert info == 0
    assert oracle.repr_error(p.Z, Q, R, m) <= 10 * n * U
    _, R0, _ = oracle.normal(p.A, p.Z, m)
    X = _sqrtA_times(p, dense(p.Z, m))
    kG = np.linalg.cond(X) ** 2
    assert np.linalg.norm(dense(R, n) - dense(R0, n)) / np.linalg.norm(dense(R0, n)) <= 10 * np.sqrt(m) * U * kG


def test_dd_orth_cols_equals_full_checker_bitwise():
    # the sampled checker is the full checker restricted to S (same per-entry arithmetic)
    p = gen.problem(333, 12, 1e4, 1e3, 8, lda=340)
    Q, _, info = oracle.normal(p.A, p.Z, p.m)
    assert info == 0
    E = oracle.dd_orth_matrix(p.A, Q, p.m)
    cols = [0, 3, 7, 11]
    Es = oracle.dd_orth_cols(p.A, Q, p.m, cols)
    assert np.array_equal(Es, E[np.ix_(cols, cols)])


# ------------------------------------------------- P2 / P5 on the paper's dense Haar V ---------
@pytest.mark.parametrize("ucase", ["random", "top", "bottom", "split"])
def test_p2_theorem1_haar(ucase):
    """sigma_i(R) = sigma_i(A^{1/2} Z) (Theorem 1) on the s7 construction with a
    dense random V: A^{1/2} = V diag(sqrt d) V^T exactly from the generator's factors."""
    m, n = 80, 10
    p = gen.problem_haar(m, n, 1e6, 1e3, 11, ucase)
    _, R, info = oracle.normal(p.A, p.Z, m)
    assert info == 0
    Zd, Ad = dense(p.Z, m), dense(p.A, m)
    X = p.V @ (np.sqrt(p.d)[:, None] * (p.V.T @ Zd))
    sx = svals(X)
    sr = svals(dense(R, n))
    # the Gram error is ~ sqrt(m) u ||M||, M = |Z|^T|A||Z| (eq.mult1-2); case 1 cancels in A Z, so
    # relative to ||G|| = sigma_1(X)^2 it carries the factor ||M|| / sigma_1(X)^2
    canc = np.linalg.norm(np.abs(Zd).T @ np.abs(Ad) @ np.abs(Zd), 2) / sx[0] ** 2
    assert np.all(np.abs(sr - sx) / sx <= 10 * np.sqrt(m) * U * canc * (sx[0] / sx) ** 2)


def test_p5_haar_closed_forms():
    """Case 2 constant ||A|| ||Q||^2 = 10^{54/79} at kappa(A) = 1e6 (golden), case 1/3
    constant kappa(A), case 5 R = I, on the dense-V construction."""
    g = GOLDEN["case2_orth_constant"]
    m, n, ka = g["m"], g["n"], g["kappa_a"]
    p = gen.problem_haar(m, n, ka, 1e2, 12, "top")
    Q, _, info = oracle.normal(p.A, p.Z, m)
    assert info == 0
    assert abs(np.log10(np.linalg.norm(dense(Q, m), 2) ** 2 * p.d[0]) - g["normA_normQ2_log10"]) < 1e-9
    for ucase in ("bottom", "split"):
        p = gen.problem_haar(m, n, ka, 1e2, 13, ucase)
        Q, _, info = oracle.normal(p.A, p.Z, m)
        assert info == 0
        # computed Q carries CHOLQR's forward error ~ u kappa(A^{1/2} Z)^2 ||M|| / ||G|| ~ 1e-6 here
        assert abs(np.linalg.norm(dense(Q, m), 2) ** 2 * p.d[0] / ka - 1.0) < 1e-4
    p = gen.problem_haar(m, n, 1e8, 1.0, 14, "aorth")
    Q, R, info = oracle.normal(p.A, p.Z, m)
    assert info == 0
    assert np.abs(dense(R, n) - np.eye(n)).max() <= 10 * m * U * 1e8
