"""Small, ragged shapes through every kernel (for compute-sanitizer memcheck/racecheck/synccheck).
    compute-sanitizer --tool memcheck python tools/sanitize_driver.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import gen  # noqa: E402
import paper_1401_5171_b200 as oqr  # noqa: E402

shapes = [(200, 10, 0), (333, 21, 1), (517, 240, 0), (130, 57, 2), (1000, 100, 8), (96, 96, 0), (640, 40, 1)]
for m, n, pad in shapes:
    p = gen.problem(m, n, 1e3, 1e2, 5, lda=m + pad)
    A = torch.from_numpy(p.A).cuda()
    Z = torch.from_numpy(p.Z).cuda()
    for v in ("normal", "normal2", "prequr"):
        Q, R, st = oqr.VARIANTS[v](A, Z)
        assert st == 0, (m, n, v, st)
    G = oqr.gram(A, Z)
    Ge = oqr.gram_euclid(Z, m=m)
    R, info = oqr.potrf(G)
    Q = oqr.trsm(Z, R, m=m)
torch.cuda.synchronize()
print("sanitize driver ok")
