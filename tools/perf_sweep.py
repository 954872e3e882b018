"""The paper's performance experiments (s8) on the B200 through the C ABI:
normalised GFLOP/s versus n for dense A at m = 10000 (normalisation 2m^2n + 2mn^2) and tridiagonal
A at m = 100000 (normalisation 2mn^2), every variant; time = minimum of 10 runs,
CUDA events around the synchronous call.  Writes a CSV.

    python tools/perf_sweep.py [out.csv]
"""
import csv
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import gen  # noqa: E402
import paper_1401_5171_b200 as oqr  # noqa: E402

out = sys.argv[1] if len(sys.argv) > 1 else "perf_sweep.csv"
NS = [10, 20, 40, 60, 80, 100, 120, 160, 200, 240]
rows = []


def min_time(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    best = float("inf")
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e-3)
    return best


m = 10000
pA = gen.problem(m, 1, 1e3, 1.0, 0x5EED)
A = torch.from_numpy(pA.A).cuda()
for n in NS:
    p = gen.problem(m, n, 1e3, 1e2, 0x5EED + n, with_A=False)
    Z = torch.from_numpy(p.Z).cuda()
    Q = torch.empty((n, m), dtype=torch.float64, device="cuda")
    R = torch.empty((n, n), dtype=torch.float64, device="cuda")
    fl = 2.0 * m * m * n + 2.0 * m * n * n
    for fam, variants in (("dense", oqr.VARIANTS), ("sym", oqr.VARIANTS_SYM)):
        for v, fn in variants.items():
            t = min_time(lambda: fn(A, Z, Q, R))
            rows.append(dict(A="dense" if fam == "dense" else "dense (sym family)", m=m, n=n, variant=v,
                             seconds=t, gflops=fl / t / 1e9))
            print(rows[-1], flush=True)
del A
m = 100000
d, e = gen.tridiag(m, 1e3)
dg, eg = torch.from_numpy(d).cuda(), torch.from_numpy(e).cuda()
for n in NS:
    p = gen.problem(m, n, 1e3, 1e2, 0x5EED + n, with_A=False)
    Z = torch.from_numpy(p.Z).cuda()
    Q = torch.empty((n, m), dtype=torch.float64, device="cuda")
    R = torch.empty((n, n), dtype=torch.float64, device="cuda")
    fl = 2.0 * m * n * n
    for v, fn in oqr.VARIANTS_TRIDIAG.items():
        t = min_time(lambda: fn(dg, eg, Z, Q, R))
        rows.append(dict(A="tridiagonal", m=m, n=n, variant=v, seconds=t, gflops=fl / t / 1e9))
        print(rows[-1], flush=True)
with open(out, "w", newline="") as f:
    w = csv.DictWriter(f, fieldnames=["A", "m", "n", "variant", "seconds", "gflops"])
    w.writeheader()
    w.writerows(rows)
print("wrote", out)
