"""Time the fused Gram kernel K1 (liboqr timing hook, CUDA events on the launching stream).

    [OQR_LIB=...] python tools/time_k1.py m n [reps] [sym]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import gen  # noqa: E402
import paper_1401_5171_b200 as oqr  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 19968
n = int(sys.argv[2]) if len(sys.argv) > 2 else 200
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
p = gen.problem(m, n, 1e3, 1e2, 1234, with_A=False)
A = torch.randn(m, m, dtype=torch.float64, device="cuda")   # timing only: values irrelevant
Z = torch.from_numpy(p.Z).cuda()
sym = len(sys.argv) > 4 and sys.argv[4] == "sym"
gram = oqr.gram_sym if sym else oqr.gram
gram(A, Z)
torch.cuda.synchronize()
oqr.timing_enable(True)
oqr.timing_reset()
for _ in range(reps):
    gram(A, Z)
ms, k, tot = oqr.timing_read()
fl = (1.0 if sym else 2.0) * m * m * n   # sym: actual work ~ m^2 n (block-lower triangle)
print(f"{os.path.basename(oqr.LIB_PATH)} m={m} n={n} {'sym' if sym else 'dense'}: K1 {ms / k:.3f} ms  "
      f"{fl / (ms / k) / 1e9:.1f} TF/s of actual work, dense-equivalent {2.0 * m * m * n / (ms / k) / 1e9:.1f}")
