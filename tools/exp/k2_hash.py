"""Hash of K2's R (oqr_potrf) for a bitwise A/B between library builds, plus its time."""
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_1401_5171_b200 as oqr  # noqa: E402

for n in [9, 50, 100, 200, 233, 240]:
    g = torch.Generator().manual_seed(n)
    X = torch.randn(n, 2 * n, dtype=torch.float64, generator=g)
    G = (X @ X.T + 0.01 * torch.eye(n, dtype=torch.float64)).cuda().contiguous()
    for _ in range(3):
        R, info = oqr.potrf(G)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        oqr.potrf(G)
    e1.record()
    torch.cuda.synchronize()
    print(n, int(info.item()), hashlib.sha256(R.cpu().numpy().tobytes()).hexdigest()[:16], f"{e0.elapsed_time(e1) / 20 * 1e3:.1f} us")
