"""The paper's s7 stability sweep through the GPU C ABI on the paper's own
construction (dense random V = orth(randn(m)), W = orth(randn(n)); gen.problem_haar): cases 1-5
(case 4: random Z), m = 80, n = 10, kappa(A) = 10^1..10^15, kappa(Z) = kappa(A)^{1/2}, variants
normal / normal2 / prequr / prequr_hh (Householder pre-step).  Errors are formed in numpy long
double (80-bit; not the test oracle).  Writes a CSV and prints per-case slope fits of
log10 ||Q^T A Q - I||_2 against log10 kappa(A).

    python tools/stability_sweep.py [out.csv]
"""
import csv
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import gen  # noqa: E402
import paper_1401_5171_b200 as oqr  # noqa: E402

M, N = 80, 10
CASES = {f"case{k}": u for k, u in gen.PAPER_CASES.items()}
VARIANTS = ("normal", "normal2", "prequr", "prequr_hh")
out = sys.argv[1] if len(sys.argv) > 1 else "stability_sweep.csv"
rows = []
for case, ucase in CASES.items():
    for variant in VARIANTS:
        for e in range(1, 16):
            ka = 10.0 ** e
            p = gen.problem_haar(M, N, ka, math.sqrt(ka), 7, ucase)
            Q, R, st = oqr.VARIANTS[variant](torch.from_numpy(p.A).cuda(), torch.from_numpy(p.Z).cuda())
            row = dict(case=case, variant=variant, kappa_A=ka, kappa_Z=math.sqrt(ka), status=st)
            if st == 0:
                Ad = p.A[:, :M].T.astype(np.longdouble)
                Zd = p.Z[:, :M].T.astype(np.longdouble)
                Qd = Q.cpu().numpy()[:, :M].T.astype(np.longdouble)
                Rd = R.cpu().numpy().T.astype(np.longdouble)
                E = (Qd.T @ (Ad @ Qd) - np.eye(N, dtype=np.longdouble)).astype(np.float64)
                D = (Zd - Qd @ Rd).astype(np.float64)
                row.update(orth=np.linalg.norm(E, 2),
                           repr=np.linalg.norm(D, 2) / np.linalg.norm(Zd.astype(np.float64), 2),
                           normA_normQ2=float(np.max(p.d)) * np.linalg.norm(Qd.astype(np.float64), 2) ** 2)
            rows.append(row)
with open(out, "w", newline="") as f:
    w = csv.DictWriter(f, fieldnames=["case", "variant", "kappa_A", "kappa_Z", "status", "orth", "repr",
                                      "normA_normQ2"])
    w.writeheader()
    for r in rows:
        w.writerow(r)
for case in CASES:
    for variant in VARIANTS:
        rr = [r for r in rows if r["case"] == case and r["variant"] == variant and r["status"] == 0
              and r["orth"] < 1e-2]
        if len(rr) >= 3:
            s = np.polyfit([math.log10(r["kappa_A"]) for r in rr], [math.log10(r["orth"]) for r in rr], 1)[0]
        else:
            s = float("nan")
        brk = [int(math.log10(r["kappa_A"])) for r in rows if r["case"] == case and r["variant"] == variant
               and r["status"] != 0]
        reps = [r["repr"] for r in rows if r["case"] == case and r["variant"] == variant and r["status"] == 0]
        print(f"{case} {variant:8s} orth slope vs log kappa(A) = {s:5.2f}  max repr = {max(reps):.2e}  "
              f"breakdown at kappa(A)=1e{brk}")
print("wrote", out)
