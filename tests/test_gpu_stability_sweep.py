"""the paper's s7 stability experiment through the GPU C ABI.

m = 80, n = 10, kappa(A) = 10^1 .. 10^15, kappa(Z) = kappa(A)^{1/2}; cases 1, 2,
3, 5 (eigenvector alignment from gen).  Errors are formed with the
oracle's double-double checkers.  The paper's claims checked here:
  * representativity ||Z - QR|| / ||Z|| is ~1e-15 and flat in kappa for every variant (Fig. repres);
  * CHOLQR's loss of orthogonality is proportional to kappa(Z)^2 in case 2 (slope 1 vs kappa(A));
  * the stable variants' loss of orthogonality is O(u ||A|| ||Q||^2) (Thm 3), i.e. kappa(A) in
    cases 1, 3 and 5 (slope 1) and flat in case 2;
  * case 5 (Z A-orthogonal): all variants show the same error.
"""
import math

import numpy as np
import pytest

import gen
import oracle
from oracle import U

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

M, N = 80, 10
EXPS = list(range(1, 16))
CASES = {"case1": "bottom", "case2": "top", "case3": "split", "case5": "aorth"}


def run_sweep(ucase, variant):
    import paper_1401_5171_b200 as oqr
    rows = []
    for e in EXPS:
        ka = 10.0 ** e
        p = gen.problem(M, N, ka, math.sqrt(ka), 7, ucase=ucase)
        Q, R, st = oqr.VARIANTS[variant](torch.from_numpy(p.A).cuda(), torch.from_numpy(p.Z).cuda())
        if st != 0:
            rows.append(dict(e=e, st=st))
            continue
        Qg, Rg = Q.cpu().numpy(), R.cpu().numpy()
        normQ = np.linalg.norm(oracle.from_cm(Qg, M), 2)
        rows.append(dict(e=e, st=0, orth=oracle.orth_error(p.A, Qg, M), rep=oracle.repr_error(p.Z, Qg, Rg, M),
                         scale=U * float(np.max(p.d)) * normQ ** 2))
    return rows


@pytest.fixture(scope="module")
def sweeps():
    return {(c, v): run_sweep(u, v) for c, u in CASES.items() for v in ("normal", "normal2", "prequr")}


def ok(rows):
    return [r for r in rows if r["st"] == 0]


def test_representativity_flat_1e15(sweeps):
    for key, rows in sweeps.items():
        reps = [r["rep"] for r in ok(rows)]
        assert reps, key
        assert max(reps) <= 1e-14, (key, max(reps))


def test_cholqr_case2_orth_proportional_to_kappaZ_squared(sweeps):
    rows = [r for r in ok(sweeps[("case2", "normal")]) if r["orth"] < 1e-3 and r["e"] >= 2]
    assert len(rows) >= 6
    slope = np.polyfit([r["e"] for r in rows], [math.log10(r["orth"]) for r in rows], 1)[0]
    assert 0.8 <= slope <= 1.2, slope          # kappa(Z)^2 = kappa(A)


@pytest.mark.parametrize("variant", ["normal2", "prequr"])
def test_stable_variants_orth_proportional_to_A_Q2(sweeps, variant):
    for case in ("case1", "case3", "case5"):
        rows = [r for r in ok(sweeps[(case, variant)]) if r["orth"] < 1e-2]
        assert len(rows) >= 8, (case, variant)
        for r in rows:
            assert r["orth"] <= 10 * N * r["scale"], (case, r)
        slope = np.polyfit([r["e"] for r in rows], [math.log10(r["orth"]) for r in rows], 1)[0]
        assert 0.7 <= slope <= 1.3, (case, variant, slope)     # ||A|| ||Q||^2 = kappa(A)
    rows = ok(sweeps[("case2", variant)])
    assert max(r["orth"] for r in rows) <= 1e-13            # best case: sigma_1/sigma_n small


def test_case5_all_variants_same_error(sweeps):
    for e in EXPS:
        vals = [r["orth"] for v in ("normal", "normal2", "prequr") for r in sweeps[("case5", v)]
                if r["e"] == e and r["st"] == 0]
        if len(vals) == 3 and min(vals) > 0:
            assert max(vals) / min(vals) <= 30.0, (e, vals)
