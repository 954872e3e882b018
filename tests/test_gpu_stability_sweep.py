"""the paper's s7 stability experiment through the GPU C ABI, on the paper's own
construction: A = V diag(d) V^T with V = orth(randn(m)) (dense, Haar), Z = U
diag(s) W^T with W = orth(randn(n)) and U the case's eigenvectors of A (cases 1, 2, 3, 5,
PAPER.md:723-740) or orth(randn(m, n)) (case 4, random Z); m = 80, n = 10,
kappa(A) = 10^1 .. 10^15, kappa(Z) = kappa(A)^{1/2}.  Errors are formed with the oracle's
double-double checkers; the bounds with tests/paper_bounds.py (c = 1).  Checked:
  * Fig. repres: ||Z - QR|| / ||Z|| ~1e-15, flat in kappa, for every variant and case, and below
    Theorem 2's componentwise bound (CHOLQR) / Theorem 3's bound (PRE-CHOLQR, repeated CHOLQR);
  * Fig. orth: CHOLQR's loss of orthogonality is below Theorem 2's eq.(orth1) at every point and
    proportional to kappa(Z)^2 in case 2 (slope 1 against kappa(A)); the stable variants
    (repeated CHOLQR, PRE-CHOLQR with the Cholesky-QR and the Householder pre-step) stay below
    Theorem 3's m n^2 u ||A|| ||Q||^2 at every point and track u ||A|| ||Q||^2: slope 1 in cases 1,
    3, 5 (||A|| ||Q||^2 = kappa(A)), flat in case 2, and within [1e-3, 10 n] of it in case 4;
  * case 5 (Z A-orthogonal): all variants show the same error;
  * Fig. repres-vs-comp: CHOLQR on case 3 with kappa(Z) = 10: the true
    error and the componentwise bound stay flat while the normwise bound grows as kappa(A)^{1/2}.
"""
import math

import numpy as np
import pytest

import gen
import oracle
import paper_bounds as pb
from gates import gate
from oracle import U

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

M, N = 80, 10
EXPS = list(range(1, 16))
CASES = {f"case{k}": u for k, u in gen.PAPER_CASES.items()}
VARIANTS = ("normal", "normal2", "prequr", "prequr_hh")


def run_point(oqr, p, variant):
    Q, R, st = oqr.VARIANTS[variant](torch.from_numpy(p.A).cuda(), torch.from_numpy(p.Z).cuda())
    row = dict(e=round(math.log10(p.kappa_a)), st=st)
    if st != 0:
        return row
    Qg, Rg = Q.cpu().numpy(), R.cpu().numpy()
    A, Z = oracle.from_cm(p.A, M), oracle.from_cm(p.Z, M)
    Qd, Rd = oracle.from_cm(Qg, M), oracle.from_cm(Rg, N)
    normA = float(np.max(p.d))
    row.update(orth=oracle.orth_error(p.A, Qg, M), rep=oracle.repr_error(p.Z, Qg, Rg, M),
               rho=oracle.componentwise_ratio(p.Z, Qg, Rg, M),
               scale=U * normA * np.linalg.norm(Qd, 2) ** 2,
               thm2=pb.thm2(A, Z, Qd, Rd, normA), thm3=pb.thm3(M, N, Qd, Rd, Z, normA))
    return row


@pytest.fixture(scope="module")
def sweeps():
    import paper_1401_5171_b200 as oqr
    out = {}
    for c, u in CASES.items():
        probs = [gen.problem_haar(M, N, 10.0 ** e, 10.0 ** (e / 2), 7, u) for e in EXPS]
        for v in VARIANTS:
            out[(c, v)] = [run_point(oqr, p, v) for p in probs]
    return out


def ok(rows):
    return [r for r in rows if r["st"] == 0]


def test_every_point_within_the_theorems(sweeps):
    for (case, v), rows in sweeps.items():
        assert ok(rows), (case, v)
        for r in ok(rows):
            tag = f"{case}/{v} kA=1e{r['e']}"
            gate("sweep repr flat ~1e-15", r["rep"], 1e-14, tag)
            if v == "normal":
                gate("sweep Thm2 comp rho", r["rho"], oracle.gamma(N + 1), tag)
                gate("sweep Thm2 orth1", r["orth"], r["thm2"]["orth1"], tag)
            else:
                gate(f"sweep Thm3 repr ({v})", r["rep"], r["thm3"]["repr_norm"], tag)
                gate(f"sweep Thm3 orth ({v})", r["orth"], r["thm3"]["orth"], tag)


def test_prequr_hh_never_breaks_down_in_the_sweep(sweeps):
    # the Householder pre-step is stable for every kappa(Z) <= 1e7.5 here; the A-stage Gram has
    # kappa ~ ||A|| ||Q||^2 <= 1e15, so PRE-CHOLQR as Algorithm 2 states it completes everywhere
    for case in CASES:
        assert all(r["st"] == 0 for r in sweeps[(case, "prequr_hh")]), case


def test_cholqr_case2_orth_proportional_to_kappaZ_squared(sweeps):
    rows = [r for r in ok(sweeps[("case2", "normal")]) if r["orth"] < 1e-3 and r["e"] >= 2]
    assert len(rows) >= 6
    s = pb.slope([10.0 ** r["e"] for r in rows], [r["orth"] for r in rows])
    assert 0.8 <= s <= 1.2, s          # kappa(Z)^2 = kappa(A)


@pytest.mark.parametrize("variant", ["normal2", "prequr", "prequr_hh"])
def test_stable_variants_track_A_Q2(sweeps, variant):
    for case in ("case1", "case3", "case5"):
        rows = [r for r in ok(sweeps[(case, variant)]) if r["orth"] < 1e-2]
        assert len(rows) >= 8, (case, variant)
        for r in rows:
            gate(f"sweep orth <= 10 n u||A||||Q||^2 ({variant})", r["orth"], 10 * N * r["scale"], f"{case} 1e{r['e']}")
        s = pb.slope([10.0 ** r["e"] for r in rows], [r["orth"] for r in rows])
        assert 0.7 <= s <= 1.3, (case, variant, s)     # ||A|| ||Q||^2 = kappa(A)
    rows = ok(sweeps[("case2", variant)])
    assert max(r["orth"] for r in rows) <= 1e-13            # best case: sigma_1/sigma_n small
    rows = ok(sweeps[("case4", variant)])                    # random Z: descriptive both ways
    assert len(rows) >= 10
    for r in rows:
        assert 1e-3 * r["scale"] <= r["orth"] <= 10 * N * r["scale"], (variant, r["e"], r["orth"] / r["scale"])


def test_case5_all_variants_same_error(sweeps):
    for e in EXPS:
        vals = [r["orth"] for v in VARIANTS for r in sweeps[("case5", v)] if r["e"] == e and r["st"] == 0]
        if len(vals) == len(VARIANTS) and min(vals) > 0:
            assert max(vals) / min(vals) <= 30.0, (e, vals)


def test_repres_vs_comp_case3():
    """Fig. repres-vs-comp: CHOLQR, case 3, kappa(Z) = 10."""
    import paper_1401_5171_b200 as oqr
    rows = []
    for e in EXPS:
        p = gen.problem_haar(M, N, 10.0 ** e, 10.0, 7, "split")
        r = run_point(oqr, p, "normal")
        if r["st"] == 0:
            rows.append(r)
    assert len(rows) >= 10
    ka = [10.0 ** r["e"] for r in rows]
    true = [r["rep"] for r in rows]
    comp = [r["thm2"]["repr_comp"] for r in rows]
    norm = [r["thm2"]["repr_norm"] for r in rows]
    for r, t, c in zip(rows, true, comp):
        gate("repres-vs-comp true <= comp bound", t, c, f"1e{r['e']}")
    assert max(true) / min(true) <= 100.0                 # true error: flat
    assert abs(pb.slope(ka, comp)) <= 0.1                 # componentwise bound: flat
    s = pb.slope(ka, norm)
    assert 0.4 <= s <= 0.6, s                             # normwise bound ~ kappa(A)^{1/2}
