"""K2 phase timeline from an OQR_EXP_POTRF_TRACE build:
    OQR_LIB=tools/exp/liboqr_k2trace.so python tools/exp/k2_trace.py [n]"""
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
buf = (ctypes.c_longlong * 256)()
assert oqr.lib().oqr_exp_k2_trace(buf) == 0
t0 = buf[0]
NT = (n + 7) // 8
print(f"n={n}: staged -> loop end {buf[1] - t0} clk, end {buf[2] - t0} clk (1965 MHz: {(buf[2] - t0) / 1965:.1f} us)")
prev = t0
for j in range(NT):
    a, b, c = buf[4 + 3 * j] - t0, buf[5 + 3 * j] - t0, (buf[6 + 3 * j] - t0) if j + 1 < NT else 0
    print(f"step {j:2d}: diag ready {a:7d}  row solved {b:7d} (+{b - a:5d})  next diag factored (warp 0) {c:7d} (+{c - b if c else 0:5d})  step {a - prev:6d}")
    prev = a
