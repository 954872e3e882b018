"""Hash of K3's Q (oqr_trsm and the full oqr_normal) for a bitwise A/B between library builds."""
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import gen  # noqa: E402
import paper_1401_5171_b200 as oqr  # noqa: E402

for m, n in [(4000, 50), (40000, 200), (1031, 9), (517, 240)]:
    p = gen.problem(m, n, 1.0, 1e2, 1234, with_A=False)
    Z = torch.from_numpy(p.Z).cuda()
    R = torch.from_numpy(np.ascontiguousarray(np.triu(np.eye(n) + 0.01 * np.ones((n, n))).T)).cuda()
    Q = oqr.trsm(Z, R, m=m)
    torch.cuda.synchronize()
    print(m, n, hashlib.sha256(Q.cpu().numpy().tobytes()).hexdigest()[:16])
