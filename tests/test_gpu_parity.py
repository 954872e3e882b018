"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the same seeded
inputs.  Gates T1-T8 of SURVEY.md s8(c) / DESIGN.md s5, each tolerance derived from the
paper's error model with c = 1:

  T1 Gram        |G_gpu - G_orc| <= 2 gamma_{3m} |Z|^T|A||Z|        (eq.mult1-2, any sum order)
  T2 repr.       rho_gpu = max |Z-QR| / (|Q||R|) <= gamma_{n+1}      (Thm 2 componentwise)
  T3 Cholesky    |G - R^T R| <= gamma_{n+1} |R|^T|R|                 (eq:normal:chol)
  T4 trsm        rho(Z, Q, R) <= gamma_{n+1} for given (Z, R)
  T5 orth.       E_gpu <= 10 E_orc + 10 n u ||A|| ||Q_orc||^2        (Thms 2-3)
  T6 forward     first-order perturbation bounds: with the two sides' Gram and
                 Cholesky errors dG = 2 gamma_{3m} |Z|^T|A||Z| + 2 gamma_{n+1} |R|^T|R|,
                 ||R_gpu - R_orc||_F <= sqrt(2) kappa(G) ||R|| ||dG||_F / ||G||   (Sun's bound, x2)
                 ||Q_gpu - Q_orc||_F <= ||Q|| ||R^-1|| tol_R + 2 gamma_{n+1} || |Q||R| ||_F ||R^-1||
  T7 outcome     same status class (0 / first Cholesky / second Cholesky)
  T8 determinism two runs bitwise equal
"""
import math

import numpy as np
import pytest

import gen
import oracle
from gates import branch, gate
from oracle import U, gamma

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def oqr():
    import paper_1401_5171_b200 as m
    m.lib()
    return m


DEV = "cuda:0"


def to_dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


# shapes spanning several 64-row panels and 16-column k-blocks, ragged tails, n not a multiple
# of 8, n = 1, n = m, n = OQR_NMAX, padded leading dimensions.
SHAPES = [
    # (m, n, kappa_A, kappa_Z, seed, lda_pad, ldz_pad)
    (200, 10, 1e2, 1e2, gen.SEED_BASE + 0, 0, 0),      # config 0
    (333, 21, 1e3, 1e2, 11, 0, 0),                      # ragged panel + ragged k-block (odd m)
    (1000, 100, 1e2, 1e2, 12, 8, 3),                    # padded lda / odd ldz
    (640, 40, 1e2, 1e3, 16, 1, 0),                      # odd lda: plain-load path for every tile
    (1031, 1, 1e4, 1.0, 13, 2, 0),                      # n = 1, m prime
    (96, 96, 1e2, 1e2, 14, 0, 0),                       # n = m
    (517, 240, 1e2, 1e2, 15, 0, 0),                     # n = OQR_NMAX, ragged
    (4000, 50, 1e4, 1e3, gen.SEED_BASE + 1, 0, 0),      # config 1
]


def make(m, n, ka, kz, seed, lda_pad=0, ldz_pad=0, ucase="reflect"):
    return gen.problem(m, n, ka, kz, seed, ucase=ucase, lda=m + lda_pad, ldz=m + ldz_pad)


def forward_tols(p, Go, Ro, Qo):
    """T6 tolerances (absolute Frobenius) for R and Q from the first-order Cholesky perturbation
    bound (Sun 1991: ||dR||_F / ||R||_2 <= kappa_2(G) ||dG||_F / (sqrt(2) ||G||_2)) applied to the
    componentwise Gram error of eq.mult1-2 and the Cholesky backward error of eq:normal:chol
    (PAPER.md:190-196), with a factor 2 for higher-order terms; Q = Z R^{-1} adds the
    substitution error of PAPER.md:197-198 on each side."""
    m, n = p.m, p.n
    Ad = np.abs(oracle.from_cm(p.A, m))
    Zd = np.abs(oracle.from_cm(p.Z, m))
    M = Zd.T @ (Ad @ Zd)
    Rd = oracle.from_cm(Ro, n)
    Qd = oracle.from_cm(Qo, m)
    dG = np.linalg.norm(2 * gamma(3 * m) * M + 2 * gamma(n + 1) * (np.abs(Rd).T @ np.abs(Rd)))
    sG = np.linalg.svd(Go, compute_uv=False)
    sR = np.linalg.svd(Rd, compute_uv=False)
    tol_R = math.sqrt(2) * (sG[0] / sG[-1]) * sR[0] * dG / sG[0]
    tol_Q = (np.linalg.norm(Qd, 2) * tol_R + 2 * gamma(n + 1) * np.linalg.norm(np.abs(Qd) @ np.abs(Rd))) / sR[-1]
    return tol_R, tol_Q


def check_gram(oqr, p):
    m = p.m
    G = host(oqr.gram(to_dev(p.A), to_dev(p.Z)))
    Gd, M = oracle.dd_gram(p.A, p.Z, m)       # dense n x n, double-double G and |Z|^T|A||Z|
    Go = oracle.from_cm(oracle.gram(p.A, p.Z, m), p.n)
    Gg = G.T                                  # storage (n, n) col-major -> dense
    tag = f"m={m} n={p.n}"
    gate("T1 |G-G_orc|/M", np.max(np.abs(Gg - Go) / M), 2 * gamma(3 * m), tag)
    gate("T1 |G-G_dd|/M", np.max(np.abs(Gg - Gd) / M), gamma(3 * m), tag)
    return G


@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: f"m{s[0]}n{s[1]}")
def test_t1_gram(oqr, shape):
    check_gram(oqr, make(*shape))


@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: f"m{s[0]}n{s[1]}")
def test_t1_gram_euclid(oqr, shape):
    p = make(*shape)
    m, n = p.m, p.n
    G = host(oqr.gram_euclid(to_dev(p.Z), m=m)).T
    Go = oracle.from_cm(oracle.gram_euclid(p.Z, m), n)
    Zd = oracle.from_cm(p.Z, m)
    M = np.abs(Zd).T @ np.abs(Zd)
    gate("T1 euclid |G-G_orc|/M", np.max(np.abs(G - Go) / M), 2 * gamma(3 * m), f"m={m} n={n}")


@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: f"m{s[0]}n{s[1]}")
def test_t3_potrf(oqr, shape):
    p = make(*shape)
    n = p.n
    G = oracle.gram(p.A, p.Z, p.m)            # oracle G (storage (n, n))
    R, info = oqr.potrf(to_dev(G))
    assert int(host(info)[0]) == 0
    Rg = host(R)
    ratio = oracle.chol_backward_ratio(oracle.from_cm(G, n), Rg)
    gate("T3 |G-RtR|/(|R|t|R|)", ratio, gamma(n + 1), f"m={p.m} n={n}")
    Ro, io = oracle.potrf(G)
    assert io == 0
    assert np.all(np.tril(oracle.from_cm(Rg, n), -1) == 0)
    # same G on both sides: only the two Cholesky backward errors differ (Sun's bound, x2)
    Rd = oracle.from_cm(Ro, n)
    dG = np.linalg.norm(2 * gamma(n + 1) * (np.abs(Rd).T @ np.abs(Rd)))
    sG = np.linalg.svd(oracle.from_cm(G, n), compute_uv=False)
    tol = math.sqrt(2) * (sG[0] / sG[-1]) * np.linalg.norm(Rd, 2) * dG / sG[0]
    gate("T3 ||R-R_orc|| (same G)", np.linalg.norm(Rg - Ro), tol, f"m={p.m} n={n}")


@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: f"m{s[0]}n{s[1]}")
def test_t4_trsm(oqr, shape):
    p = make(*shape)
    m, n = p.m, p.n
    R, _ = oracle.potrf(oracle.gram(p.A, p.Z, m))
    Q = host(oqr.trsm(to_dev(p.Z), to_dev(R), m=m))
    rho = oracle.componentwise_ratio(p.Z, Q, R, m)
    gate("T4 rho (trsm)", rho, gamma(n + 1), f"m={m} n={n}")
    Qo = oracle.trsm(p.Z, R, m)
    # same (Z, R): each side's substitution error |dR^i| <= gamma_n |R|
    Rd, Qd = oracle.from_cm(R, n), oracle.from_cm(Qo, m)
    sR = np.linalg.svd(Rd, compute_uv=False)
    tol = 2 * gamma(n + 1) * np.linalg.norm(np.abs(Qd) @ np.abs(Rd)) / sR[-1]
    gate("T4 ||Q-Q_orc|| (same Z, R)", np.linalg.norm(Q - Qo), tol, f"m={m} n={n}")


def test_potrf_breakdown_examples(oqr):
    # [[1,2],[2,1]] breaks down at pivot 2; NaN pivot breaks down (reading R4)
    G = oracle.to_cm(np.array([[1.0, 2.0], [2.0, 1.0]]))
    _, info = oqr.potrf(to_dev(G))
    assert int(host(info)[0]) == 2
    G = np.eye(3)
    G[1, 1] = np.nan
    _, info = oqr.potrf(to_dev(oracle.to_cm(G)))
    assert int(host(info)[0]) == 2
    G = oracle.to_cm(np.array([[4.0, 2.0], [2.0, 5.0]]))
    R, info = oqr.potrf(to_dev(G))
    assert int(host(info)[0]) == 0
    assert np.array_equal(oracle.from_cm(host(R), 2), np.array([[2.0, 1.0], [0.0, 2.0]]))


def _certain_success(A, Zc, m, n, euclid=False):
    """True when every Cholesky of G = Z^T A Z computed with ANY summation order completes:
    lambda_min(G) exceeds 10x the first-order bound on the Gram error, gamma_{3m} ||M||_2
    (eq.mult1-2), plus Cholesky's own n^2 u ||G|| (completion condition,
    PAPER.md:200-201).  Otherwise the outcome (success or the breakdown pivot) is decided by
    rounding and is not a parity criterion (parity unpinned)."""
    if euclid:
        Zd = oracle.from_cm(Zc, m)
        G = Zd.T @ Zd
        M = np.abs(Zd).T @ np.abs(Zd)
    else:
        G, M = oracle.dd_gram(A, Zc, m)
    lam = np.linalg.eigvalsh((G + G.T) / 2)
    err = gamma(3 * m) * np.linalg.norm(M, 2) + n * n * U * lam[-1]
    return lam[0] > 10 * err


def outcome_determined(p, variant):
    m, n = p.m, p.n
    if variant == "prequr_stable":   # stable pre-step: only the A-stage can break down
        Y, _, info = oracle.scqr3(p.Z, m)
        return info == 0 and _certain_success(p.A, Y, m, n)
    if variant == "prequr_hh":       # Householder pre-step never breaks down
        Y, _ = oracle.hhqr(p.Z, m)
        return _certain_success(p.A, Y, m, n)
    if variant in ("normal", "normal2"):
        ok = _certain_success(p.A, p.Z, m, n)
        if ok and variant == "normal2":
            Q1, _, st1 = oracle.normal(p.A, p.Z, m)
            ok = st1 == 0 and _certain_success(p.A, Q1, m, n)
        return ok
    ok = _certain_success(None, p.Z, m, n, euclid=True)
    if ok:
        S, _ = oracle.potrf(oracle.gram_euclid(p.Z, m))
        Y = oracle.trsm(p.Z, S, m)
        ok = _certain_success(p.A, Y, m, n)
    return ok


def _nrm(X):
    return float(np.linalg.norm(X, 2))


def cholqr_orth_bound(A, Z, Q, R, normA):
    """Theorem 2, eq. (orth1) with c = 1, for one CHOLQR pass on (A, Z) with
    computed factors (Q, R) (dense matrices):
    ||Q^T A Q - I|| <= m n u ||R^-1|| ||Z|| (||R^-1|| ||A Z|| + ||Q|| ||A||)."""
    m, n = Z.shape
    smin = np.linalg.svd(R, compute_uv=False)[-1]
    if smin == 0:
        return math.inf
    return m * n * U * _nrm(Z) / smin * (_nrm(A @ Z) / smin + _nrm(Q) * normA)


def thm3_orth_bound(m, n, Q, normA):
    """Theorem 3 with c = 1: ||Q^T A Q - I|| <= m n^2 u ||Q||^2 ||A||."""
    return m * n * n * U * _nrm(Q) ** 2 * normA


def decompose(oqr, fam, variant, A_dev, Z_dev, m):
    """The intermediate factors of a GPU variant, recomputed through the library's own step
    exports and oqr_normal: normal2 = two CHOLQR passes (Q1, R1), (Q, R2); prequr = the Euclidean
    pre-step (Y, S) and the A-stage (Q, U).  The variant runs exactly these kernels, so the
    recomputed Q must equal the variant's Q bitwise (asserted by the caller)."""
    nrm = fam["normal"]
    if variant == "normal2":
        Q1, R1, s1 = nrm(A_dev, Z_dev)
        assert s1 == 0
        Q, R2, s2 = nrm(A_dev, Q1)
        return dict(Z1=Q1, F1=R1, Q=Q, F2=R2, st=s2)
    if variant == "prequr":
        G = oqr.gram_euclid(Z_dev, m=m)
        S, info = oqr.potrf(G)
        assert int(host(info)[0]) == 0
        Y = oqr.trsm(Z_dev, S, m=m)
        Q, U_, s2 = nrm(A_dev, Y)
        return dict(Z1=Y, F1=S, Q=Q, F2=U_, st=s2)
    if variant == "prequr_hh":
        Y, S = oqr.hhqr(Z_dev, m=m)
        Q, U_, s2 = nrm(A_dev, Y)
        return dict(Z1=Y, F1=S, Q=Q, F2=U_, st=s2)
    return None


def theorem_gates(oqr, fam, p, variant, Qg, Rg, A_dev, Z_dev, tag):
    """Theorems 2 and 3 on the GPU's own factors (no oracle result needed), for every variant:
      normal        |Z - QR| <= gamma_{n+1} |Q||R|; eq.(orth1)                       (Thm 2)
      normal2       Thm 2 on each of its two CHOLQR passes, eq.(orth1) for the second;
                    R = R2 R1 to the product's rounding (2 gamma_n |R2||R1|)
      prequr(_hh)   |Z - QR| <= m n^2 u |Q||U||S|; ||Q^T A Q - I|| <= m n^2 u ||Q||^2 ||A||; R = U S (Thm 3)
      prequr_stable |Z - QR| <= m n^2 u |Q||R| (sufficient for Thm 3's form); Thm 3 orthogonality
    with the paper's constant c = 1."""
    m, n = p.m, p.n
    Rd, Qd = oracle.from_cm(Rg, n), oracle.from_cm(Qg, m)
    assert np.all(np.isfinite(Qd)) and np.all(np.isfinite(Rd))
    assert np.all(np.tril(Rd, -1) == 0) and np.all(np.diag(Rd) > 0)
    A = oracle.from_cm(p.A, m)
    Z = oracle.from_cm(p.Z, m)
    normA = float(np.max(p.d))
    E = oracle.orth_error(p.A, Qg, m)
    if variant == "normal":
        gate("Thm2 rho (normal)", oracle.componentwise_ratio(p.Z, Qg, Rg, m), gamma(n + 1), tag)
        gate("Thm2 orth1 (normal)", E, cholqr_orth_bound(A, Z, Qd, Rd, normA), tag)
        return
    if variant == "prequr_stable":
        gate("Thm3 rho (prequr_stable)", oracle.componentwise_ratio(p.Z, Qg, Rg, m), m * n * n * U, tag)
        gate("Thm3 orth (prequr_stable)", E, thm3_orth_bound(m, n, Qd, normA), tag)
        return
    dec = decompose(oqr, fam, variant, A_dev, Z_dev, m)
    assert dec["st"] == 0 and np.array_equal(host(dec["Q"]), Qg), "intermediate factors do not reproduce Q"
    Z1 = host(dec["Z1"])
    F1, F2 = oracle.from_cm(host(dec["F1"]), n), oracle.from_cm(host(dec["F2"]), n)
    gate(f"Thm R=F2*F1 ({variant})", np.max(np.abs(Rd - F2 @ F1) / (np.abs(F2) @ np.abs(F1) + 1e-300)),
         2 * gamma(n), tag)
    if variant == "normal2":
        gate("Thm2 rho pass1 (normal2)", oracle.componentwise_ratio(p.Z, Z1, host(dec["F1"]), m), gamma(n + 1), tag)
        gate("Thm2 rho pass2 (normal2)", oracle.componentwise_ratio(Z1, Qg, host(dec["F2"]), m), gamma(n + 1), tag)
        gate("Thm2 orth1 pass2 (normal2)", E, cholqr_orth_bound(A, oracle.from_cm(Z1, m), Qd, F2, normA), tag)
    else:
        D, _ = oracle.dd_resid(p.Z, Qg, Rg, m)
        QUS = np.abs(Qd) @ np.abs(F2) @ np.abs(F1)
        mask = QUS > U * np.abs(Z).max()
        gate(f"Thm3 |Z-QR|/(|Q||U||S|) ({variant})", float((np.abs(D)[mask] / QUS[mask]).max()) if mask.any() else 0.0,
             m * n * n * U, tag)
        gate(f"Thm3 orth ({variant})", E, thm3_orth_bound(m, n, Qd, normA), tag)


def kappa_t6(p, variant, Go):
    """kappa_2 of the Gram matrix whose perturbation sets the forward error of R: G = Z^T A Z for
    CHOLQR; for the pre-QR variants also the pre-step's Z^T Z (the Euclidean Cholesky-QR pre-step's S
    carries u kappa(Z)^2 relative error)."""
    sG = np.linalg.svd(Go, compute_uv=False)
    k = sG[0] / sG[-1] if sG[-1] > 0 else math.inf
    if variant.startswith("prequr"):
        sZ = np.linalg.svd(oracle.from_cm(p.Z, p.m), compute_uv=False)
        k = max(k, (sZ[0] / sZ[-1]) ** 2)
    return k


def variant_gates(oqr, p, variant, family="dense"):
    m, n = p.m, p.n
    fams = {"dense": oqr.VARIANTS, "sym": oqr.VARIANTS_SYM,
            # oqr_normal_host: host arrays in and out, A staged in 64- or 128-column chunks
            "host64": {"normal": lambda A, Z: oqr.normal_host(A.cpu(), Z.cpu(), chunk_cols=64)},
            "host128": {"normal": lambda A, Z: oqr.normal_host(A.cpu().pin_memory(), Z.cpu().pin_memory(),
                                                               chunk_cols=128)},
            "host": {"normal": lambda A, Z: oqr.normal_host(A.cpu().pin_memory(), Z.cpu())}}
    fam = fams[family]
    tag = f"{family}/{variant} m={m} n={n} kA={p.kappa_a:.0e} kZ={p.kappa_z:.0e} {p.ucase}"
    A_dev, Z_dev = to_dev(p.A), to_dev(p.Z)
    Q, R, st = fam[variant](A_dev, Z_dev)
    Qo, Ro, sto = oracle.VARIANTS[variant](p.A, p.Z, m)
    cls = lambda s: 0 if s == 0 else (1 if s <= n else 2)
    assert 0 <= st <= 2 * n and 0 <= sto <= 2 * n, (st, sto)
    determined = outcome_determined(p, variant)
    if determined:                                              # T7
        assert st == 0 and sto == 0, (st, sto)
    if st != 0:
        # breakdown where rounding decides the outcome (reading R20): a valid result, counted
        branch(f"T7 undetermined, GPU breakdown class {cls(st)}, oracle class {cls(sto)}")
        return None
    Qg, Rg = host(Q), host(R)
    theorem_gates(oqr, fam, p, variant, Qg, Rg, A_dev, Z_dev, tag)
    if sto != 0:
        # GPU success where the oracle broke down (rounding-decided): the theorems above are the
        # paper's whole claim about such a result; there is no oracle factor to compare with
        branch(f"T7 undetermined, GPU success, oracle class {cls(sto)} ({variant}): Thm 2/3 gates only")
        return Qg, Rg, st
    branch(f"both succeed ({'determined' if determined else 'undetermined'})")
    rho = oracle.componentwise_ratio(p.Z, Qg, Rg, m)           # T2
    rho_o = oracle.componentwise_ratio(p.Z, Qo, Ro, m)
    if variant == "normal":
        gate("T2 rho (normal)", rho, gamma(n + 1), tag)
    else:
        gate(f"T2 rho vs oracle ({variant})", rho, 10 * rho_o + 4 * gamma(n + 1), tag)
    e = oracle.orth_error(p.A, Qg, m)                          # T5
    eo = oracle.orth_error(p.A, Qo, m)
    normA = float(np.max(p.d))                                  # ||A||_2 (generator ground truth)
    normQ = np.linalg.norm(oracle.from_cm(Qo, m), 2)
    tol = 10 * eo + 10 * n * U * normA * normQ ** 2
    if variant == "normal":
        A, Z = oracle.from_cm(p.A, m), oracle.from_cm(p.Z, m)
        tol = max(tol, cholqr_orth_bound(A, Z, oracle.from_cm(Qo, m), oracle.from_cm(Ro, n), normA))
    gate(f"T5 orth ({variant})", e, tol, tag)
    G = oracle.from_cm(oracle.gram(p.A, p.Z, m), n)             # T6
    tol_R, tol_Q = forward_tols(p, G, Ro, Qo)
    dR, dQ = np.linalg.norm(Rg - Ro), np.linalg.norm(Qg - Qo)
    gate(f"T6 R first-order ({variant})", dR, tol_R, tag)
    gate(f"T6 Q first-order ({variant})", dQ, tol_Q, tag)
    # the survey's probabilistic gate sqrt(m) u kappa(G), relative Frobenius.
    # It assumes ||Delta G|| ~ sqrt(m) u ||G||, which holds for the generator's configs (no
    # cancellation in Z^T A Z).  The s7 constructions (eigenvector-aligned Z, kappa(A) up to 1e10)
    # cancel: Delta G ~ sqrt(m) u |Z|^T|A||Z| >> u ||G||, so there the same first-order estimate
    # carries the factor ||M||_2 / ||G||_2 (M = |Z|^T|A||Z|, eq.mult1-2).
    k6 = kappa_t6(p, variant, G)
    t6 = math.sqrt(m) * U * k6
    if p.ucase != "reflect":
        Ad, Zd = np.abs(oracle.from_cm(p.A, m)), np.abs(oracle.from_cm(p.Z, m))
        t6 *= max(1.0, np.linalg.norm(Zd.T @ (Ad @ Zd), 2) / np.linalg.norm(G, 2))
    gate(f"T6s R sqrt(m)u kappa ({variant})", dR / np.linalg.norm(Ro), t6, tag)
    gate(f"T6s Q sqrt(m)u kappa ({variant})", dQ / np.linalg.norm(Qo), t6, tag)
    return Qg, Rg, st


@pytest.mark.parametrize("variant", ["normal", "normal2", "prequr", "prequr_stable", "prequr_hh"])
@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: f"m{s[0]}n{s[1]}")
def test_t2_t5_t6_t7_variants(oqr, shape, variant):
    variant_gates(oqr, make(*shape), variant)


@pytest.mark.parametrize("variant", ["normal", "normal2", "prequr"])
def test_t8_determinism(oqr, variant):
    p = make(4000, 50, 1e4, 1e3, 99)
    A, Z = to_dev(p.A), to_dev(p.Z)
    Q1, R1, s1 = oqr.VARIANTS[variant](A, Z)
    Q2, R2, s2 = oqr.VARIANTS[variant](A, Z)
    assert s1 == s2 == 0
    assert torch.equal(Q1, Q2) and torch.equal(R1, R2)
    G1 = oqr.gram(A, Z)
    G2 = oqr.gram(A, Z)
    assert torch.equal(G1, G2)


@pytest.mark.parametrize("ucase", ["top", "bottom", "split", "aorth"])
def test_paper_cases_small(oqr, ucase):
    # the paper's s7 constructions at m = 80, n = 10
    for ka in (1e2, 1e6, 1e10):
        p = gen.problem(80, 10, ka, math.sqrt(ka), 5, ucase=ucase)
        for v in ("normal", "normal2", "prequr", "prequr_hh"):
            variant_gates(oqr, p, v)


def test_breakdown_witness_small(oqr):
    # paper case 3 with kappa(A^{1/2}Z)^2 = kappa(G) = 1e20 >> 1/u: CHOLQR must break down in its
    # (first) Cholesky, normal2 in pass 1; prequr still succeeds (s8(c) item 14)
    p = gen.problem(400, 20, 1e8, 1e6, 77, ucase="split")
    A, Z = to_dev(p.A), to_dev(p.Z)
    _, _, st = oqr.normal(A, Z)
    _, _, sto = oracle.normal(p.A, p.Z, p.m)
    assert 1 <= st <= p.n and 1 <= sto <= p.n
    _, _, st2 = oqr.normal2(A, Z)
    assert 1 <= st2 <= p.n
    variant_gates(oqr, p, "prequr")


def test_nan_input_breaks_down(oqr):
    p = make(300, 12, 1e2, 1e2, 3)
    Z = p.Z.copy()
    Z[4, 17] = np.nan
    _, _, st = oqr.normal(to_dev(p.A), to_dev(Z))
    assert 1 <= st <= p.n


def test_abi_argument_errors_on_device(oqr):
    p = make(64, 8, 1e2, 1e2, 1)
    A, Z = to_dev(p.A), to_dev(p.Z)
    Q = torch.empty((8, 64), dtype=torch.float64, device=DEV)
    R = torch.empty((8, 8), dtype=torch.float64, device=DEV)
    import ctypes
    L = oqr.lib()
    P = ctypes.c_void_p
    s = P(torch.cuda.current_stream().cuda_stream)
    assert L.oqr_normal(64, 8, P(A.data_ptr() + 4), 64, P(Z.data_ptr()), 64, P(Q.data_ptr()), P(R.data_ptr()), s) == -3
    assert L.oqr_normal(64, 8, P(A.data_ptr()), 64, P(Z.data_ptr()), 64, P(Q.data_ptr()), P(R.data_ptr()), s) == 0


def test_stream_and_launch_accounting(oqr):
    p = make(500, 30, 1e2, 1e2, 2)
    A, Z = to_dev(p.A), to_dev(p.Z)
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        n0 = oqr.launch_count()
        Q, R, s = oqr.normal(A, Z)
        assert s == 0
        assert oqr.launch_count() - n0 == 5          # pack, K1, K1r, K2, K3
    Qo, Ro, _ = oracle.normal(p.A, p.Z, p.m)
    assert np.linalg.norm(host(R) - Ro) / np.linalg.norm(Ro) < 1e-12


# ---------------------------------------------------- NEXT-N4: symmetric A (block-lower triangle)
@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: f"m{s[0]}n{s[1]}")
def test_t1_gram_sym(oqr, shape):
    p = make(*shape)
    m, n = p.m, p.n
    G = host(oqr.gram_sym(to_dev(p.A), to_dev(p.Z)))
    assert np.array_equal(G, G.T)                                   # bitwise symmetric by construction
    Gd, M = oracle.dd_gram(p.A, p.Z, m)
    Go = oracle.from_cm(oracle.gram(p.A, p.Z, m), n)
    assert np.all(np.abs(G.T - Go) <= 2 * gamma(3 * m) * M)
    assert np.all(np.abs(G.T - Gd) <= gamma(3 * m) * M)


@pytest.mark.parametrize("variant", ["normal", "normal2", "prequr", "prequr_hh"])
@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: f"m{s[0]}n{s[1]}")
def test_variants_sym(oqr, shape, variant):
    variant_gates(oqr, make(*shape), variant, family="sym")


def test_sym_reads_only_block_lower_triangle(oqr):
    # poisoning the strictly block-upper part of A must not change the result
    p = make(300, 20, 1e3, 1e2, 17)
    A = p.A.copy()                  # storage (cols, rows): A[j, i] is element (i, j)
    for j in range(300):
        for i in range(300):
            if j // 64 > i // 64:   # block column beyond the row's block: upper, never read
                A[j, i] = np.nan
    Q1, R1, s1 = oqr.normal_sym(to_dev(p.A), to_dev(p.Z))
    Q2, R2, s2 = oqr.normal_sym(to_dev(A), to_dev(p.Z))
    assert s1 == s2 == 0
    assert torch.equal(R1, R2) and torch.equal(Q1, Q2)


def test_sym_determinism(oqr):
    p = make(4000, 50, 1e4, 1e3, 99)
    A, Z = to_dev(p.A), to_dev(p.Z)
    G1, G2 = oqr.gram_sym(A, Z), oqr.gram_sym(A, Z)
    assert torch.equal(G1, G2)


def test_upload_sym_copies_what_sym_reads(oqr):
    p = make(333, 21, 1e3, 1e2, 23)
    A_h = torch.from_numpy(p.A)                       # (m, lda) column-major host A
    A_d = torch.full_like(A_h, float("nan"), device=DEV)
    oqr.upload_sym(A_h, A_d)
    torch.cuda.synchronize()
    Q1, R1, s1 = oqr.normal_sym(A_d, to_dev(p.Z))
    Q2, R2, s2 = oqr.normal_sym(to_dev(p.A), to_dev(p.Z))
    assert s1 == s2 == 0 and torch.equal(R1, R2) and torch.equal(Q1, Q2)


# ---------------------------------------------------- NEXT-N1: stable pre-step (shifted CholeskyQR3)
@pytest.mark.parametrize("kz", [1e8, 1e10, 1e12])
def test_prequr_stable_ill_conditioned_Z(oqr, kz):
    """kappa(Z) beyond the Euclidean Cholesky-QR pre-step's limit (reading R2): oqr_prequr breaks
    down in its pre-step (kappa >= 1e10), oqr_prequr_stable succeeds with Theorem 3's orthogonality
    and matches the oracle (gates T2, T5, T6, T7)."""
    p = gen.problem(2000, 40, 1e6, kz, 61)
    if kz >= 1e10:
        _, _, st = oqr.prequr(to_dev(p.A), to_dev(p.Z))
        assert 1 <= st <= p.n
    r = variant_gates(oqr, p, "prequr_stable")
    assert r is not None
    Qg = r[0]
    E = oracle.orth_error(p.A, Qg, p.m)
    scale = U * float(np.max(p.d)) * np.linalg.norm(oracle.from_cm(Qg, p.m), 2) ** 2
    assert E <= 10 * p.n * scale


def test_prequr_stable_beyond_its_range(oqr):
    # shifted CholeskyQR3 is stable for kappa(Z) <~ 1/(11 (m n + n(n+1)) u) (~1e10..1e12 here);
    # at 1e14 kappa(Q1) ~ 1e9 > u^{-1/2}, so the CholeskyQR2 stage's Gram has kappa ~ 1e18 > 1/u
    # and whether its Cholesky breaks down is decided by rounding (reading R20: parity
    # unpinned).  Pinned: the oracle breaks down; a GPU success must still return an upper
    # triangular R with a positive diagonal and finite Q; a GPU breakdown is a first-stage code.
    p = gen.problem(2000, 40, 1e6, 1e14, 61)
    Q, R, st = oqr.prequr_stable(to_dev(p.A), to_dev(p.Z))
    _, _, sto = oracle.prequr_stable(p.A, p.Z, p.m)
    assert 1 <= sto <= p.n
    assert 0 <= st <= p.n
    if st == 0:
        Rd = oracle.from_cm(host(R), p.n)
        assert np.all(np.tril(Rd, -1) == 0) and np.all(np.diag(Rd) > 0)
        assert np.all(np.isfinite(host(Q)))


@pytest.mark.parametrize("family", ["sym", "tridiag"])
def test_prequr_stable_families(oqr, family):
    if family == "sym":
        p = gen.problem(1000, 30, 1e4, 1e11, 62)
        Q, R, st = oqr.prequr_stable_sym(to_dev(p.A), to_dev(p.Z))
        Qo, Ro, sto = oracle.prequr_stable(p.A, p.Z, p.m)
        A_orth = lambda Q: oracle.orth_error(p.A, Q, p.m)
    else:
        d, e = gen.tridiag(3000, 1e4)
        p = gen.problem(3000, 30, 1e4, 1e11, 63, with_A=False)
        Q, R, st = oqr.prequr_stable_tridiag(torch.from_numpy(d).cuda(), torch.from_numpy(e).cuda(), to_dev(p.Z))
        Qo, Ro, sto = oracle.prequr_stable(oracle.densify_tridiag(d, e), p.Z, p.m)
        A_orth = lambda Q: oracle.orth_error_tridiag(d, e, Q, p.m)
    assert st == 0 and sto == 0
    Qg, Rg = host(Q), host(R)
    assert A_orth(Qg) <= 10 * A_orth(Qo) + 1e-12
    assert oracle.componentwise_ratio(p.Z, Qg, Rg, p.m) <= 10 * oracle.componentwise_ratio(p.Z, Qo, Ro, p.m) + 4 * gamma(p.n + 1)


@pytest.mark.parametrize("variant", ["normal", "normal2", "prequr", "prequr_stable", "prequr_hh"])
@pytest.mark.parametrize("mn", [(1, 1), (2, 2), (3, 1), (7, 3), (8, 8), (64, 64), (65, 1)])
def test_tiny_shapes(oqr, variant, mn):
    # the 64 x KS tensor-TMA box exceeds the whole matrix: rows/cols beyond m are zero-filled
    m, n = mn
    p = gen.problem(m, n, 10.0, 10.0, 81, lda=m + (m & 1))
    Q, R, st = oqr.VARIANTS[variant](to_dev(p.A), to_dev(p.Z))
    Qo, Ro, sto = oracle.VARIANTS[variant](p.A, p.Z, m)
    assert st == sto == 0
    Qg, Rg = host(Q), host(R)
    assert np.allclose(Rg, Ro, rtol=1e-12, atol=1e-14 * np.abs(Ro).max())
    assert np.allclose(Qg, Qo, rtol=1e-10, atol=1e-12 * np.abs(Qo).max())
    if variant == "normal":
        assert oracle.componentwise_ratio(p.Z, Qg, Rg, m) <= gamma(n + 1)
    Gs = host(oqr.gram_sym(to_dev(p.A), to_dev(p.Z))).T
    Go = oracle.from_cm(oracle.gram(p.A, p.Z, m), n)
    Zd = np.abs(oracle.from_cm(p.Z, m))
    M = Zd.T @ (np.abs(oracle.from_cm(p.A, m)) @ Zd)
    assert np.all(np.abs(Gs - Go) <= 2 * gamma(3 * m) * M)


# oqr_normal_host: the same CHOLQR on host arrays, A moved in column chunks with the Gram of each
# chunk accumulated into the same slots (include/oqr.h).  Gates T2/T5/T6/T7 against the oracle
# for several chunk sizes (64: a chunk per k-block group, ragged last chunk; auto = m/8), T8.
@pytest.mark.parametrize("family", ["host64", "host128", "host"])
@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: f"m{s[0]}n{s[1]}")
def test_normal_host(oqr, shape, family):
    variant_gates(oqr, make(*shape), "normal", family)


def test_normal_host_determinism_and_gram(oqr):
    p = make(4000, 50, 1e4, 1e3, 99, 3, 1)
    Ah, Zh = torch.from_numpy(p.A).pin_memory(), torch.from_numpy(p.Z)
    Q1, R1, s1 = oqr.normal_host(Ah, Zh, chunk_cols=192)
    Q2, R2, s2 = oqr.normal_host(Ah, Zh, chunk_cols=192)
    assert s1 == s2 == 0 and torch.equal(Q1, Q2) and torch.equal(R1, R2)                     # T8
    # T3 on the chunked Gram: R^T R reproduces the oracle's G within eq.mult1-2 + eq:normal:chol
    m, n = p.m, p.n
    Go = oracle.from_cm(oracle.gram(p.A, p.Z, m), n)
    Rd = R1.numpy().T
    Ad, Zd = np.abs(oracle.from_cm(p.A, m)), np.abs(oracle.from_cm(p.Z, m))
    M = Zd.T @ (Ad @ Zd)
    assert np.all(np.abs(Rd.T @ Rd - Go) <= 2 * gamma(3 * m) * M + 2 * gamma(n + 1) * (np.abs(Rd).T @ np.abs(Rd)))


def test_normal_host_argument_errors(oqr):
    import ctypes
    L = oqr.lib()
    A = torch.zeros((64, 64), dtype=torch.float64)
    Z = torch.zeros((8, 64), dtype=torch.float64)
    Q = torch.zeros((8, 64), dtype=torch.float64)
    R = torch.zeros((8, 8), dtype=torch.float64)
    P = lambda t: ctypes.c_void_p(t.data_ptr())
    s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    assert L.oqr_normal_host(64, 8, None, 64, P(Z), 64, P(Q), P(R), 0, s) == -3
    assert L.oqr_normal_host(64, 8, P(A), 63, P(Z), 64, P(Q), P(R), 0, s) == -4
    assert L.oqr_normal_host(64, 8, P(A), 64, P(Z), 64, P(Q), P(R), -1, s) == -9
    assert L.oqr_normal_host(64, 65, P(A), 64, P(Z), 64, P(Q), P(R), 0, s) == -2


# K4 family (upper triangle by tile-row pairs): one CTA part per K-slice up to NT = 18, two from
# NT = 19 (n > 144), three from NT = 27 (n > 208); quotas of 2..8 units per warp change with NT.
# n on both sides of those boundaries and of the widest shapes, Euclidean and tridiagonal Grams
# (T1; the mirrored lower triangle must equal the upper bitwise).
@pytest.mark.parametrize("n", [40, 41, 48, 49, 88, 89, 96, 97, 144, 145, 208, 209, 232, 233, 240])
def test_t1_packed_upper_gram_part_boundaries(oqr, n):
    m = 1000 + n
    p = make(m, n, 1e2, 1e2, 70 + n)
    Z = to_dev(p.Z)
    G = host(oqr.gram_euclid(Z, m=m)).T
    assert np.array_equal(G, G.T)
    Go = oracle.from_cm(oracle.gram_euclid(p.Z, m), n)
    Zd = oracle.from_cm(p.Z, m)
    assert np.all(np.abs(G - Go) <= 2 * gamma(3 * m) * (np.abs(Zd).T @ np.abs(Zd)))
    d, e = gen.tridiag(m, 1e3)
    Gt = host(oqr.gram_tridiag(to_dev(d), to_dev(e), Z)).T
    assert np.array_equal(Gt, Gt.T)
    Got = oracle.from_cm(oracle.gram_tridiag(d, e, p.Z, m), n)
    Td = np.abs(np.diag(d)) + np.abs(np.diag(e, 1)) + np.abs(np.diag(e, -1))
    Mt = np.abs(Zd).T @ (Td @ np.abs(Zd))
    assert np.all(np.abs(Gt - Got) <= 2 * gamma(m + 3) * Mt)


@pytest.mark.parametrize("m,n", [(1000, 1), (1031, 9), (517, 50), (3001, 145), (2003, 200), (2003, 209),
                                 (777, 240), (40000, 200)])
def test_euclid_box_gram_bitwise_packed_path(oqr, m, n):
    """K4e (the Euclidean Gram reading the column-major Z once by tensor TMA, 20-row boxes) against
    the packed path an odd ldz selects (Zp through HBM, then K4'): the same products in the same
    order per tile and the same K-slices, so G is bitwise equal; both within T1 of the oracle."""
    p = gen.problem(m, n, 1e2, 1e2, 91 + n, with_A=False)
    Zev = torch.full((n, m + (m & 1)), float("nan"), dtype=torch.float64)
    Zev[:, :m] = torch.from_numpy(p.Z)
    Zodd = torch.full((n, m + (1 if m % 2 == 0 else 2)), float("nan"), dtype=torch.float64)
    Zodd[:, :m] = torch.from_numpy(p.Z)
    G1 = oqr.gram_euclid(Zev.cuda(), m=m)
    G2 = oqr.gram_euclid(Zodd.cuda(), m=m)
    assert torch.equal(G1, G2)
    G = host(G1).T
    assert np.array_equal(G, G.T)
    if m * n <= 2e6:
        Go = oracle.from_cm(oracle.gram_euclid(p.Z, m), n)
        Zd = oracle.from_cm(p.Z, m)
        gate("T1 euclid box |G-G_orc|/M", np.max(np.abs(G - Go) / (np.abs(Zd).T @ np.abs(Zd))), 2 * gamma(3 * m),
             f"m={m} n={n}")


def test_timing_hook_per_kernel(oqr):
    """oqr_timing_read_kernel: one K1, K2, K3 launch per oqr_normal; prequr adds the packed Gram
    (K4') and a second K2/K3; the K1 reading equals oqr_timing_read's."""
    p = make(2000, 30, 1e2, 1e2, 81)
    A, Z = to_dev(p.A), to_dev(p.Z)
    oqr.timing_enable(True)
    try:
        oqr.timing_reset()
        oqr.normal(A, Z)
        counts = {k: oqr.timing_read_kernel(k)[1] for k in ("K1", "K4", "K3", "K2")}
        assert counts == {"K1": 1, "K4": 0, "K3": 1, "K2": 1}, counts
        ms, k1, _ = oqr.timing_read()
        assert k1 == 1 and ms == oqr.timing_read_kernel("K1")[0] and ms > 0
        oqr.timing_reset()
        oqr.prequr(A, Z)
        counts = {k: oqr.timing_read_kernel(k)[1] for k in ("K1", "K4", "K3", "K2")}
        assert counts == {"K1": 1, "K4": 1, "K3": 2, "K2": 2}, counts
    finally:
        oqr.timing_enable(False)


# The paper's dense construction (V = orth(randn(m)), U random: case 4) at moderate sizes: Z is not
# aligned with a few coordinate directions, so every row of A and Z carries weight (round-1
# advice: the 4-reflector configs concentrate Z in its leading n x n block).
HAAR = [(2000, 40, 1e4, 1e3, 101, 0), (2001, 100, 1e6, 1e2, 102, 3), (1500, 240, 1e2, 1e2, 103, 1)]
_HAAR_CACHE = {}


@pytest.mark.parametrize("variant", ["normal", "normal2", "prequr", "prequr_stable", "prequr_hh"])
@pytest.mark.parametrize("hp", HAAR, ids=lambda h: f"m{h[0]}n{h[1]}")
def test_variants_haar_random(oqr, hp, variant):
    m, n, ka, kz, seed, pad = hp
    if hp not in _HAAR_CACHE:   # O(m^3) construction: once per shape
        _HAAR_CACHE[hp] = gen.problem_haar(m, n, ka, kz, seed, "random", lda=m + pad, ldz=m + pad)
    p = _HAAR_CACHE[hp]
    variant_gates(oqr, p, variant)
    if variant == "normal":
        check_gram(oqr, p)
