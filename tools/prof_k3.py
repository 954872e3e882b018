"""Small driver for ncu: K3 (oqr_trsm, Q = Z R^{-1}) at (m, n) `reps` times on a well-conditioned R.

    python tools/prof_k3.py [m] [n] [reps]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import gen  # noqa: E402
import paper_1401_5171_b200 as oqr  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 40000
n = int(sys.argv[2]) if len(sys.argv) > 2 else 200
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
p = gen.problem(m, n, 1.0, 1e2, 1234, with_A=False)
Z = torch.from_numpy(p.Z).cuda()
R = torch.from_numpy(np.ascontiguousarray(np.triu(np.eye(n) + 0.01 * np.ones((n, n))).T)).cuda()
for _ in range(reps):
    oqr.trsm(Z, R, m=m)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(10):
    oqr.trsm(Z, R, m=m)
e.record()
torch.cuda.synchronize()
print(f"ok trsm m={m} n={n}: {s.elapsed_time(e) / 10:.4f} ms")
