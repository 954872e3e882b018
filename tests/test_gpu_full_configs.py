"""GPU parity at BASELINE.json's FULL sizes (configs[2], configs[3], configs[4] and the configs[4]
breakdown witness), through the same C-ABI calls bench.py times (oqr_normal / oqr_normal2 /
oqr_prequr on device-resident inputs).

Checked against the CPU oracle on the same seeded inputs:
  * T1: every entry of G = Z^T A Z within 2 gamma_{3m} (|Z|^T|A||Z|)  (eq.mult1-2)
  * T7: outcome class (the witness must break down for normal / normal2 and not for prequr)
  * T2: componentwise representativity on ALL of Q, R (double-double residual, O(mn^2))
  * T5: orthogonality on a column subset S (all n columns at c4 and the witness, 44 at c2, 22 at
        c3, always the first/last three and the rest spread evenly): Q_S^T A Q_S - I in
        double-double, against 10 E_orc + 10 n u ||A|| ||Q_orc||^2 on the same S, and Theorem 3's
        m n^2 u ||Q||^2 ||A|| for the pre-QR / repeated variants
  * T6: R and Q against the oracle's, first-order perturbation tolerances (test_gpu_parity)
  * T8: bitwise determinism of two calls
"""
import math

import numpy as np
import pytest

import gen
import oracle
from gates import gate
from oracle import U, gamma

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

DEV = "cuda:0"


def absA_absZ(p):
    """M = |Z|^T |A| |Z| in FP64 (a tolerance scale, not a parity value), blockwise over A."""
    m = p.m
    Zd = np.abs(oracle.from_cm(p.Z, m))
    AZ = np.zeros((m, p.n))
    for j0 in range(0, m, 2048):
        j1 = min(m, j0 + 2048)
        AZ += np.abs(p.A[j0:j1, :m]).T @ Zd[j0:j1]
    return Zd.T @ AZ


@pytest.fixture(scope="module", params=["c4", "witness", "c2", "c3"])
def case(request):
    import paper_1401_5171_b200 as oqr
    name = request.param
    p = gen.witness() if name == "witness" else gen.config(int(name[1]))
    A = torch.from_numpy(p.A).to(DEV)
    Z = torch.from_numpy(p.Z).to(DEV)
    d = dict(name=name, p=p, A=A, Z=Z, oqr=oqr, M=absA_absZ(p),
             G=oracle.from_cm(oracle.gram(p.A, p.Z, p.m), p.n))
    yield d
    del d["A"], d["Z"]
    torch.cuda.empty_cache()


def test_t1_gram_full(case):
    p, oqr = case["p"], case["oqr"]
    n = p.n
    Gg = oqr.gram(case["A"], case["Z"]).cpu().numpy().T
    Go = case["G"]
    tol = 2 * gamma(3 * p.m) * case["M"]
    gate("T1 full |G-G_orc|/M", np.max(np.abs(Gg - Go) / case["M"]), 2 * gamma(3 * p.m), case["name"])
    assert np.all(np.abs(Gg - Go) <= tol)


def sampled_cols(m, n):
    """All columns when the double-double check costs <= ~1e10 multiply-adds, else an even spread
    (with the first and last three, where the extreme singular directions of Z sit)."""
    k = n if m * m * n <= 1.1e10 else (48 if m * m * n <= 5e10 else 24)
    if k >= n:
        return list(range(n))
    return sorted(set([0, 1, 2, n - 3, n - 2, n - 1] + list(np.linspace(0, n - 1, k - 6).round().astype(int))))


@pytest.mark.parametrize("variant", ["normal", "normal2", "prequr", "prequr_stable", "prequr_hh", "normal_sym",
                                     "prequr_sym", "normal_host"])
def test_variants_full(case, variant):
    p, oqr = case["p"], case["oqr"]
    m, n = p.m, p.n
    if variant.endswith("_sym"):      # NEXT-N4: same mathematics, block-lower triangle of A only
        variant = variant[:-4]
        fn = oqr.VARIANTS_SYM[variant]
    elif variant == "normal_host":    # host arrays in and out, A staged in column chunks
        variant = "normal"
        Ah, Zh = torch.from_numpy(p.A), torch.from_numpy(p.Z)
        fn = lambda A, Z: oqr.normal_host(Ah, Zh)
    else:
        fn = oqr.VARIANTS[variant]
    Q, R, st = fn(case["A"], case["Z"])
    Q2, R2, st2 = fn(case["A"], case["Z"])
    assert st == st2                                                            # T8
    if st == 0:                        # on breakdown Q and R are unspecified (include/oqr.h)
        assert torch.equal(Q, Q2) and torch.equal(R, R2)
    Qo, Ro, sto = oracle.VARIANTS[variant](p.A, p.Z, m)
    cls = lambda s: 0 if s == 0 else (1 if s <= n else 2)
    if case["name"] == "witness":                                               # T7
        # kappa(A^{1/2}Z)^2 = kappa(G) = 1e20 >> 1/u: CHOLQR breaks down in its first Cholesky
        # (normal2 in pass 1); the pre-QR variant's A-stage is well conditioned (s8(c) item 14)
        expect = 0 if variant.startswith("prequr") else 1
        assert cls(st) == expect and cls(sto) == expect, (st, sto)
    else:
        assert st == 0 and sto == 0, (st, sto)
    if st != 0:
        return
    Qg, Rg = Q.cpu().numpy(), R.cpu().numpy()
    tag = f"{case['name']}/{variant}"
    rho = oracle.componentwise_ratio(p.Z, Qg, Rg, m)                            # T2
    if variant == "normal":
        gate("T2 full rho (normal)", rho, gamma(n + 1), tag)
    else:
        rho_o = oracle.componentwise_ratio(p.Z, Qo, Ro, m)
        gate(f"T2 full rho vs oracle ({variant})", rho, 10 * rho_o + 4 * gamma(n + 1), tag)
        gate(f"Thm3 full rho ({variant})", rho, m * n * n * U, tag)
    S = sampled_cols(m, n)                                                       # T5 (sampled)
    E = np.linalg.norm(oracle.dd_orth_cols(p.A, Qg, m, S), 2)
    Eo = np.linalg.norm(oracle.dd_orth_cols(p.A, Qo, m, S), 2)
    normQ = np.linalg.norm(oracle.from_cm(Qo, m), 2)
    normA = float(np.max(p.d))
    gate(f"T5 full orth |S|={len(S)} ({variant})", E, 10 * Eo + 10 * n * U * normA * normQ ** 2, tag)
    if variant != "normal":
        normQg = np.linalg.norm(oracle.from_cm(Qg, m), 2)
        gate(f"Thm3 full orth ({variant})", E, m * n * n * U * normA * normQg ** 2, tag)
    # T6: first-order perturbation bounds (see test_gpu_parity.forward_tols)
    G = case["G"]
    Rd, Qd = oracle.from_cm(Ro, n), oracle.from_cm(Qo, m)
    dG = np.linalg.norm(2 * gamma(3 * m) * case["M"] + 2 * gamma(n + 1) * (np.abs(Rd).T @ np.abs(Rd)))
    sG = np.linalg.svd(G, compute_uv=False)
    sR = np.linalg.svd(Rd, compute_uv=False)
    tol_R = math.sqrt(2) * (sG[0] / sG[-1]) * sR[0] * dG / sG[0]
    tol_Q = (np.linalg.norm(Qd, 2) * tol_R + 2 * gamma(n + 1) * np.linalg.norm(np.abs(Qd) @ np.abs(Rd))) / sR[-1]
    dR, dQ = np.linalg.norm(Rg - Ro), np.linalg.norm(Qg - Qo)
    gate(f"T6 full R first-order ({variant})", dR, tol_R, tag)
    gate(f"T6 full Q first-order ({variant})", dQ, tol_Q, tag)
    k6 = sG[0] / sG[-1]
    if variant.startswith("prequr"):
        sZ = np.linalg.svd(oracle.from_cm(p.Z, m), compute_uv=False)
        k6 = max(k6, (sZ[0] / sZ[-1]) ** 2)
    # the survey's own T6 gate: relative Frobenius error <= sqrt(m) u kappa
    gate(f"T6s full R sqrt(m)u kappa ({variant})", dR / np.linalg.norm(Ro), math.sqrt(m) * U * k6, tag)
    gate(f"T6s full Q sqrt(m)u kappa ({variant})", dQ / np.linalg.norm(Qo), math.sqrt(m) * U * k6, tag)
