"""GPU parity of the Householder pre-step (K6, oqr_hhqr) and of PRE-CHOLQR as Algorithm 2 states it
(oqr_prequr_hh), against the CPU oracle (orc_hhqr / orc_prequr_hh) on the same seeded inputs.

Householder QR's R factor is unique (positive diagonal) but its computed Y and S are not forward
stable for ill-conditioned Z: they differ from another Householder QR's by O(u kappa(Z)).  So the
gates are the properties that define a backward-stable Euclidean QR -- the ones Theorem 3
 assumes of the pre-step -- plus forward agreement to the first-order bound:
  H1  ||Y^T Y - I||_2 <= m n u                       (double-double checker)
  H2  ||Z - Y S||_2 <= m n u ||Z||_2                  (double-double residual)
  H3  S upper triangular, positive diagonal; Y, S finite
  H4  ||S - S_orc||_F <= 2 m n u kappa(Z) ||S_orc||_F and ||Y - Y_orc||_F <= 2 m n u kappa(Z) sqrt(n)
      (first-order perturbation of the QR factors, both sides' backward errors)
  H5  bitwise determinism of two calls
and for oqr_prequr_hh the variant gates of test_gpu_parity (T2/T5/T6/T7, Theorem 3) plus, at
kappa(Z) = 1e12..1e15 where the Cholesky-based pre-steps (oqr_prequr, oqr_prequr_stable) break
down, Theorem 3's orthogonality O(u ||A|| ||Q||^2) and representativity O(u).
"""
import math

import numpy as np
import pytest

import gen
import oracle
from gates import gate, note
from oracle import U

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

DEV = "cuda:0"


@pytest.fixture(scope="module")
def oqr():
    import paper_1401_5171_b200 as m
    m.lib()
    return m


def to_dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


# (m, n, kappa_Z, seed, ldz_pad): one CTA, several CTAs with ragged row blocks, n = 1, n = m,
# n = OQR_NMAX, panels of 16 with a ragged last panel, the configs' shapes, a padded ldz
HH_SHAPES = [
    (200, 10, 1e2, 1, 0),
    (333, 21, 1e6, 2, 3),
    (1031, 1, 1.0, 3, 0),
    (96, 96, 1e3, 4, 0),
    (517, 240, 1e2, 5, 0),
    (4000, 50, 1e3, 6, 0),
    (9001, 37, 1e10, 7, 1),
    (20000, 100, 1e14, 8, 0),
]


@pytest.mark.parametrize("shape", HH_SHAPES, ids=lambda s: f"m{s[0]}n{s[1]}k{s[2]:.0e}")
def test_hhqr_step(oqr, shape):
    m, n, kz, seed, pad = shape
    p = gen.problem(m, n, 1.0, kz, seed, with_A=False, ldz=m + pad)
    Zg = to_dev(p.Z)
    Y, S = oqr.hhqr(Zg, m=m)
    Y2, S2 = oqr.hhqr(Zg, m=m)
    assert torch.equal(Y, Y2) and torch.equal(S, S2)                         # H5
    Yg, Sg = host(Y), host(S)
    tag = f"m={m} n={n} kZ={kz:.0e}"
    Sd = oracle.from_cm(Sg, n)
    assert np.all(np.isfinite(Yg)) and np.all(np.isfinite(Sg))              # H3
    assert np.array_equal(Sd, np.triu(Sd)) and np.all(np.diag(Sd) > 0)
    gate("H1 ||Y^T Y - I||", oracle.orth_error_euclid(Yg, m), m * n * U, tag)
    D, _ = oracle.dd_resid(p.Z, Yg, Sg, m)
    Zd = oracle.from_cm(p.Z, m)
    gate("H2 ||Z - YS||/||Z||", np.linalg.norm(D, 2) / np.linalg.norm(Zd, 2), m * n * U, tag)
    Yo, So = oracle.hhqr(p.Z, m)
    sz = np.linalg.svd(Zd, compute_uv=False)
    kap = sz[0] / sz[-1]
    gate("H4 ||S - S_orc||/||S_orc||", np.linalg.norm(Sg - So) / np.linalg.norm(So), 2 * m * n * U * kap, tag)
    gate("H4 ||Y - Y_orc||", np.linalg.norm(Yg - Yo), 2 * m * n * U * kap * math.sqrt(n), tag)
    # the oracle's own Householder QR satisfies the same H1/H2 (sanity of the comparison)
    note("H1 oracle ||Y^T Y - I||", oracle.orth_error_euclid(Yo, m), m * n * U, tag)


def test_hhqr_identity_and_exact_cases(oqr):
    """Z = I[:, :n] (every column already reduced: tau = 0) gives Y = Z, S = I exactly; a column
    with a negative diagonal and nothing below it flips sign exactly."""
    m, n = 70, 5
    Z = np.zeros((n, m))
    for j in range(n):
        Z[j, j] = 1.0
    Y, S = oqr.hhqr(to_dev(Z), m=m)
    assert np.array_equal(host(Y), Z) and np.array_equal(host(S), np.eye(n))
    Z[2, 2] = -3.0
    Y, S = oqr.hhqr(to_dev(Z), m=m)
    Yd, Sd = host(Y), host(S)
    assert Sd[2, 2] == 3.0 and Yd[2, 2] == -1.0
    Z = np.array([[3.0, 4.0]])                      # [3; 4] -> Y = [.6; .8], S = [5]
    Y, S = oqr.hhqr(to_dev(Z), m=2)
    assert host(S)[0, 0] == 5.0
    assert np.allclose(host(Y), [[0.6, 0.8]], rtol=0, atol=2 * U)


def test_hhqr_nan_propagates(oqr):
    p = gen.problem(500, 12, 1.0, 1e2, 9, with_A=False)
    Z = p.Z.copy()
    Z[3, 100] = np.nan
    Y, S = oqr.hhqr(to_dev(Z), m=500)
    assert np.isnan(host(S)).any()


@pytest.mark.parametrize("kz", [1e12, 1e14, 1e15])
def test_prequr_hh_beyond_cholesky_prestep_range(oqr, kz):
    """kappa(Z) where the Euclidean Cholesky-QR pre-step breaks down and shifted CholeskyQR3 is at
    or past its limit: PRE-CHOLQR with the Householder pre-step succeeds on the GPU with Theorem 3's
    orthogonality and O(u) representativity, like the oracle's."""
    m, n, ka = 2000, 40, 1e6
    p = gen.problem(m, n, ka, kz, 61)
    A, Z = to_dev(p.A), to_dev(p.Z)
    _, _, st_plain = oqr.prequr(A, Z)
    assert 1 <= st_plain <= n                               # Euclidean Cholesky-QR pre-step fails
    Q, R, st = oqr.prequr_hh(A, Z)
    Qo, Ro, sto = oracle.prequr_hh(p.A, p.Z, m)
    assert st == 0 and sto == 0
    Qg, Rg = host(Q), host(R)
    tag = f"kZ={kz:.0e}"
    normA = float(np.max(p.d))
    E = oracle.orth_error(p.A, Qg, m)
    Eo = oracle.orth_error(p.A, Qo, m)
    normQ = np.linalg.norm(oracle.from_cm(Qg, m), 2)
    gate("Thm3 orth (prequr_hh, ill-cond Z)", E, m * n * n * U * normA * normQ ** 2, tag)
    gate("T5 orth vs oracle (prequr_hh, ill-cond Z)", E, 10 * Eo + 10 * n * U * normA * normQ ** 2, tag)
    gate("Thm3 repr (prequr_hh, ill-cond Z)", oracle.repr_error(p.Z, Qg, Rg, m), 10 * n * U, tag)
    _, _, st_s = oqr.prequr_stable(A, Z)
    note("prequr_stable status at this kappa(Z) (0 = success)", float(st_s), 1.0, tag)


def test_prequr_hh_families(oqr):
    """The symmetric (block-lower) and tridiagonal A-stages behind the same Householder pre-step."""
    p = gen.problem(1000, 30, 1e4, 1e13, 62)
    Q, R, st = oqr.prequr_hh_sym(to_dev(p.A), to_dev(p.Z))
    Qo, Ro, sto = oracle.prequr_hh(p.A, p.Z, p.m)
    assert st == 0 and sto == 0
    Qg = host(Q)
    normQ = np.linalg.norm(oracle.from_cm(Qg, p.m), 2)
    assert oracle.orth_error(p.A, Qg, p.m) <= 10 * oracle.orth_error(p.A, Qo, p.m) + 10 * 30 * U * normQ ** 2
    d, e = gen.tridiag(3000, 1e4)
    p = gen.problem(3000, 30, 1e4, 1e13, 63, with_A=False)
    Q, R, st = oqr.prequr_hh_tridiag(to_dev(d), to_dev(e), to_dev(p.Z))
    Qo, Ro, sto = oracle.prequr_hh(oracle.densify_tridiag(d, e), p.Z, p.m)
    assert st == 0 and sto == 0
    Qg = host(Q)
    Eg = oracle.orth_error_tridiag(d, e, Qg, p.m)
    Eo = oracle.orth_error_tridiag(d, e, Qo, p.m)
    normQ = np.linalg.norm(oracle.from_cm(Qg, p.m), 2)
    assert Eg <= 10 * Eo + 10 * 30 * U * float(d.max() + 2) * normQ ** 2


def test_prequr_hh_async_matches_sync(oqr):
    p = gen.problem(3000, 64, 1e4, 1e9, 64)
    A, Z = to_dev(p.A), to_dev(p.Z)
    Q1, R1, st = oqr.prequr_hh(A, Z)
    assert st == 0
    m, n = p.m, p.n
    ws = torch.empty(oqr.workspace_bytes(m, n), dtype=torch.uint8, device=DEV)
    status = torch.full((1,), -7, dtype=torch.int32, device=DEV)
    Q2 = torch.empty_like(Q1)
    R2 = torch.empty_like(R1)
    oqr.prequr_hh_async(A, Z, Q2, R2, ws, status)
    torch.cuda.synchronize()
    assert int(status.item()) == 0
    assert torch.equal(Q1, Q2) and torch.equal(R1, R2)
