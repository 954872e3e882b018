"""Time K2 (oqr_potrf) on a random SPD n x n G:  [OQR_LIB=...] python tools/time_potrf.py n [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1401_5171_b200 as oqr  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 200
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
g = torch.Generator().manual_seed(5)
X = torch.randn(n, 2 * n, dtype=torch.float64, generator=g)
G = (X @ X.T + n * torch.eye(n, dtype=torch.float64)).cuda().contiguous()
R, info = oqr.potrf(G)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    oqr.potrf(G, R, info)
e1.record()
torch.cuda.synchronize()
# oqr.potrf stores R column-major: the (n, n) tensor holds R^T row-wise
Rm = R.T.cpu()
Rref = torch.linalg.cholesky(G.cpu()).T
ok = bool(torch.allclose(Rm, Rref, rtol=1e-12, atol=1e-12 * float(Rref.abs().max()))) and \
    bool(torch.equal(torch.tril(Rm, -1), torch.zeros_like(Rm)))
print(f"{os.path.basename(oqr.LIB_PATH)} potrf n={n}: {e0.elapsed_time(e1) / reps * 1e3:.1f} us  info={int(info.item())}  "
      f"R^T R == G: {ok}")
