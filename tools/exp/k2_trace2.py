"""K2 per-(step, warp) phase timeline from an OQR_EXP_POTRF_TRACE2 build:
    OQR_LIB=tools/exp/liboqr_k2trace2.so python tools/exp/k2_trace2.py [n]
Per step: barrier A passed; the latest warp to finish phase 2 (row solve) and when; barrier B
passed; the latest warp to finish phase 3 (trailing tiles / warp 0's look-ahead factor)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_1401_5171_b200 as oqr  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 200
g = torch.Generator().manual_seed(5)
X = torch.randn(n, 2 * n, dtype=torch.float64, generator=g)
G = (X @ X.T + n * torch.eye(n, dtype=torch.float64)).cuda().contiguous()
for _ in range(3):
    R, info = oqr.potrf(G)
torch.cuda.synchronize()
buf = (ctypes.c_longlong * (32 * 32 * 4))()
assert oqr.lib().oqr_exp_k2_trace2(buf) == 0
NT = (n + 7) // 8
st = lambda j, w, k: buf[(j * 32 + w) * 4 + k]  # noqa: E731
t0 = st(0, 0, 0)
# only same-warp differences are used for durations (clock64 need not agree across sub-partitions);
# "skew" = spread of the barrier-A exit stamps over the warps
for j in range(NT):
    a0 = [st(j, w, 0) for w in range(32)]
    d2 = [st(j, w, 1) - st(j, w, 0) for w in range(32)]
    wB = [st(j, w, 2) - st(j, w, 1) for w in range(32)]
    d3 = [st(j, w, 3) - st(j, w, 2) for w in range(32)]
    m2 = max(range(32), key=lambda w: d2[w])
    m3 = max(range(32), key=lambda w: d3[w])
    print(f"step {j:2d}: A {st(j, 0, 0) - t0:7d} skew {max(a0) - min(a0):6d} | ph2 max w{m2:2d} {d2[m2]:5d} "
          f"median {sorted(d2)[16]:5d} | B wait w0 {wB[0]:5d} | ph3 max w{m3:2d} {d3[m3]:5d} w0 {d3[0]:5d} "
          f"median {sorted(d3)[16]:5d}")
out = os.environ.get("K2_TRACE_RAW")
if out:
    import numpy as np
    np.save(out, np.array(list(buf), dtype=np.int64).reshape(32, 32, 4))
