"""GPU parity for tridiagonal A (NEXT-N3) through the C ABI
(oqr_normal_tridiag / oqr_normal2_tridiag / oqr_prequr_tridiag / oqr_gram_tridiag) against the
tridiagonal oracle (pinned bitwise to the dense oracle in test_oracle_tridiag.py).  Gates as in
test_gpu_parity.py with the tridiagonal error scale M = |Z|^T |T| |Z| (3-term rows: gamma_{m+3})."""
import math

import numpy as np
import pytest

import gen
import oracle
from oracle import U, gamma

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def oqr():
    import paper_1401_5171_b200 as m
    m.lib()
    return m


def absT_times(d, e, X):
    Y = np.abs(d)[:, None] * np.abs(X)
    Y[:-1] += np.abs(e)[:, None] * np.abs(X[1:])
    Y[1:] += np.abs(e)[:, None] * np.abs(X[:-1])
    return Y


def problem(m, n, ka, kz, seed, ldz_pad=0):
    d, e = gen.tridiag(m, ka)
    p = gen.problem(m, n, ka, kz, seed, with_A=False, ldz=m + ldz_pad)
    return d, e, p


def gates(oqr, d, e, p, variant, check_orth=True):
    m, n = p.m, p.n
    dg, eg, Z = torch.from_numpy(d).cuda(), torch.from_numpy(e).cuda(), torch.from_numpy(p.Z).cuda()
    Q, R, st = oqr.VARIANTS_TRIDIAG[variant](dg, eg, Z)
    Q2, R2, st2 = oqr.VARIANTS_TRIDIAG[variant](dg, eg, Z)
    assert st == st2 == 0 and torch.equal(Q, Q2) and torch.equal(R, R2)            # T7, T8
    Qo, Ro, sto = oracle.VARIANTS_TRIDIAG[variant](d, e, p.Z, m)
    assert sto == 0
    Qg, Rg = Q.cpu().numpy(), R.cpu().numpy()
    rho = oracle.componentwise_ratio(p.Z, Qg, Rg, m)                               # T2
    if variant == "normal":
        assert rho <= gamma(n + 1), rho / U
    else:
        assert rho <= 10 * oracle.componentwise_ratio(p.Z, Qo, Ro, m) + 4 * gamma(n + 1)
    lam = np.linalg.eigvalsh(np.diag(d) + np.diag(e, 1) + np.diag(e, -1)) if m <= 3000 else None
    normA = lam[-1] if lam is not None else float(np.max(np.abs(d)) + 2 * np.max(np.abs(e)))
    if check_orth:                                                                  # T5
        E = oracle.orth_error_tridiag(d, e, Qg, m)
        Eo = oracle.orth_error_tridiag(d, e, Qo, m)
        normQ = np.linalg.norm(oracle.from_cm(Qo, m), 2)
        assert E <= 10 * Eo + 10 * n * U * normA * normQ ** 2, (E, Eo)
    Zd = oracle.from_cm(p.Z, m)                                                     # T6
    M = np.abs(Zd).T @ absT_times(d, e, Zd)
    G = oracle.from_cm(oracle.gram_tridiag(d, e, p.Z, m), n)
    Rd, Qd = oracle.from_cm(Ro, n), oracle.from_cm(Qo, m)
    dG = np.linalg.norm(2 * gamma(m + 3) * M + 2 * gamma(n + 1) * (np.abs(Rd).T @ np.abs(Rd)))
    sG = np.linalg.svd(G, compute_uv=False)
    sR = np.linalg.svd(Rd, compute_uv=False)
    tol_R = math.sqrt(2) * (sG[0] / sG[-1]) * sR[0] * dG / sG[0]
    tol_Q = (np.linalg.norm(Qd, 2) * tol_R + 2 * gamma(n + 1) * np.linalg.norm(np.abs(Qd) @ np.abs(Rd))) / sR[-1]
    assert np.linalg.norm(Rg - Ro) <= tol_R
    assert np.linalg.norm(Qg - Qo) <= tol_Q


SHAPES = [(2000, 30, 1e3, 1e2, 5, 0), (333, 21, 1e4, 1e2, 6, 3), (517, 240, 1e2, 1e2, 7, 0),
          (1031, 1, 1e3, 1.0, 8, 0), (96, 96, 1e2, 1e2, 9, 0), (2, 2, 10.0, 10.0, 10, 0)]


@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: f"m{s[0]}n{s[1]}")
def test_t1_gram_tridiag(oqr, shape):
    m, n, ka, kz, seed, pad = shape
    d, e, p = problem(m, n, ka, kz, seed, pad)
    G = oqr.gram_tridiag(torch.from_numpy(d).cuda(), torch.from_numpy(e).cuda(),
                         torch.from_numpy(p.Z).cuda()).cpu().numpy().T
    Go = oracle.from_cm(oracle.gram_tridiag(d, e, p.Z, m), n)
    Zd = oracle.from_cm(p.Z, m)
    M = np.abs(Zd).T @ absT_times(d, e, Zd)
    assert np.all(np.abs(G - Go) <= 2 * gamma(m + 3) * M)


@pytest.mark.parametrize("variant", ["normal", "normal2", "prequr"])
@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: f"m{s[0]}n{s[1]}")
def test_variants_tridiag(oqr, shape, variant):
    m, n, ka, kz, seed, pad = shape
    d, e, p = problem(m, n, ka, kz, seed, pad)
    gates(oqr, d, e, p, variant)


def test_eigenvector_closed_form_gpu(oqr):
    m, n, ka = 4000, 16, 1e6
    d, e = gen.tridiag(m, ka)
    ks = list(range(1, 9)) + list(range(m - 7, m + 1))
    lam, V = gen.tridiag_eigen(m, ka, ks)
    s = np.logspace(0, -3, n)
    Zc = oracle.to_cm(V * s)
    Q, R, st = oqr.normal_tridiag(torch.from_numpy(d).cuda(), torch.from_numpy(e).cuda(),
                                  torch.from_numpy(Zc).cuda())
    assert st == 0
    Rd = oracle.from_cm(R.cpu().numpy(), n)
    expect = s * np.sqrt(lam)                   # Theorem 1: R = diag(sigma(A^{1/2} Z))
    assert np.allclose(np.diag(Rd), expect, rtol=1e-9, atol=0)
    assert np.abs(np.triu(Rd, 1)).max() <= 1e-9 * expect.max()


@pytest.mark.parametrize("variant", ["normal", "normal2", "prequr"])
def test_full_size_config_T(oqr, variant):
    d, e, p = gen.tridiag_config("T")
    gates(oqr, d, e, p, variant, check_orth=(variant != "normal2"))


@pytest.mark.parametrize("m,n", [(2000, 30), (1031, 1), (517, 240), (96, 96), (16, 8), (17, 9), (3001, 145),
                                 (2003, 209), (100000, 200)])
def test_fused_stencil_gram_bitwise_packed_path(oqr, m, n):
    """K4t (Z read once by tensor TMA, stencil fused, 20-row boxes with halo) against the packed path
    (Zp and W = T Z through HBM, then K4'), which an odd ldz selects: the same W arithmetic and the
    same DMMA schedule, so G is bitwise equal wherever both use the same K-slices -- including the
    halo rows at block and CTA-slice boundaries and the first / last rows of T -- and within T1 of
    the oracle everywhere."""
    d, e = gen.tridiag(m, 1e3)
    p = gen.problem(m, n, 1e3, 1e2, 71, with_A=False)
    dg, eg = torch.from_numpy(d).cuda(), torch.from_numpy(e).cuda()
    Zev = torch.full((n, m + (m & 1)), float("nan"), dtype=torch.float64)
    Zev[:, :m] = torch.from_numpy(p.Z)                     # even ldz (16-byte aligned): the fused path
    Zev = Zev.cuda()
    Zodd = torch.full((n, m + (1 if m % 2 == 0 else 2)), float("nan"), dtype=torch.float64)
    Zodd[:, :m] = torch.from_numpy(p.Z)                    # odd ldz: the packed path
    Zodd = Zodd.cuda()
    G1 = oqr.gram_tridiag(dg, eg, Zev)
    G2 = oqr.gram_tridiag(dg, eg, Zodd)
    assert torch.equal(G1, G2)   # the same K-slices and CTA parts on both paths: bitwise
    Go = oracle.from_cm(oracle.gram_tridiag(d, e, p.Z, m), n)
    Zd = oracle.from_cm(p.Z, m)
    M = np.abs(Zd).T @ absT_times(d, e, Zd)
    assert np.all(np.abs(G1.cpu().numpy().T - Go) <= 2 * gamma(m + 3) * M)
