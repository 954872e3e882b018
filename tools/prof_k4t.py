"""Small driver for ncu: the tridiagonal Gram (oqr_gram_tridiag: K4t fused stencil when Z is
16-byte aligned with an even ldz, else pack + K4') at (m, n) `reps` times, then its event time.

    python tools/prof_k4t.py [m] [n] [reps] [packed|euclid|euclid_packed]

euclid: the Euclidean Gram oqr_gram_euclid instead (K4e box path; euclid_packed: odd ldz, pack + K4').
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import gen  # noqa: E402
import paper_1401_5171_b200 as oqr  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
n = int(sys.argv[2]) if len(sys.argv) > 2 else 200
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
mode = sys.argv[4] if len(sys.argv) > 4 else "fused"
packed = mode in ("packed", "euclid_packed")
d, e = gen.tridiag(m, 1e3)
p = gen.problem(m, n, 1e3, 1e2, 1234, with_A=False, ldz=m + (1 if packed else 0) + (m & 1 if not packed else 0))
dg, eg, Z = torch.from_numpy(d).cuda(), torch.from_numpy(e).cuda(), torch.from_numpy(p.Z).cuda()
def call():
    if mode.startswith("euclid"):
        oqr.gram_euclid(Z, m=m)
    else:
        oqr.gram_tridiag(dg, eg, Z)


for _ in range(reps):
    call()
torch.cuda.synchronize()
s, t = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(10):
    call()
t.record()
torch.cuda.synchronize()
print(f"ok {'gram_euclid' if mode.startswith('euclid') else 'gram_tridiag'} m={m} n={n} {mode}: "
      f"{s.elapsed_time(t) / 10:.4f} ms")
