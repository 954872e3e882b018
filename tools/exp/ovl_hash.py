"""Hashes of (Q, R, status) of every variant on a few shapes, repeated (graph replay from the second
call), incl. a Cholesky breakdown: a bitwise A/B between library builds (OQR_LIB), e.g. the
overlapped K2 -> K3 pair against the serial one."""
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import gen  # noqa: E402
import paper_1401_5171_b200 as oqr  # noqa: E402


def h(t):
    return hashlib.sha256(t.cpu().numpy().tobytes()).hexdigest()[:12]


for (m, n, ka, kz) in [(200, 10, 1e2, 1e2), (4000, 50, 1e3, 1e2), (1031, 9, 1e2, 1e1), (3000, 200, 1e2, 1e2),
                       (777, 232, 1e1, 1e1), (900, 240, 1e1, 1e1), (4000, 50, 1e3, 1e12)]:
    p = gen.problem(m, n, ka, kz, 77)
    A = torch.from_numpy(p.A).cuda()
    Z = torch.from_numpy(p.Z).cuda()
    for name, fn in oqr.VARIANTS.items():
        out = []
        for rep in range(3):
            Q, R, st = fn(A, Z, check=False)
            torch.cuda.synchronize()
            out.append((h(Q) if st == 0 else "-", h(R) if st == 0 else "-", st))
        assert out[0] == out[1] == out[2], (m, n, name, out)
        print(m, n, kz, name, *out[0])
    d, e = gen.tridiag(m, 1e3)
    dd, ee = torch.from_numpy(d).cuda(), torch.from_numpy(e).cuda()
    for name, fn in oqr.VARIANTS_TRIDIAG.items():
        Q, R, st = fn(dd, ee, Z, check=False)
        Q2, R2, st2 = fn(dd, ee, Z, check=False)
        torch.cuda.synchronize()
        assert (h(Q), h(R), st) == (h(Q2), h(R2), st2) or st != 0
        print(m, n, kz, "tridiag", name, h(Q) if st == 0 else "-", h(R) if st == 0 else "-", st)
print("done")
