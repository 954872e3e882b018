"""Small driver for ncu / compute-sanitizer: generate an (m, n) problem and call the step export
oqr_gram `reps` times (each call = pack_z, gram_fused (K1), gram_reduce (K1r)).

    python tools/prof_k1.py [m] [n] [reps] [variant|gram]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import gen  # noqa: E402
import paper_1401_5171_b200 as oqr  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
n = int(sys.argv[2]) if len(sys.argv) > 2 else 200
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
what = sys.argv[4] if len(sys.argv) > 4 else "gram"
p = gen.problem(m, n, 1e3, 1e2, 1234)
A = torch.from_numpy(p.A).cuda()
Z = torch.from_numpy(p.Z).cuda()
for _ in range(reps):
    if what == "gram":
        oqr.gram(A, Z)
    else:
        Q, R, st = oqr.VARIANTS[what](A, Z)
        assert st == 0, st
torch.cuda.synchronize()
print("ok", m, n, reps, what)
