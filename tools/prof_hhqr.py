"""Phase breakdown of K6 (Householder QR) from an experiment build with -DOQR_EXP_HH_PROF:
CTA 0's %globaltimer stamps at the phase boundaries.

    OQR_LIB=tools/exp/liboqr_HHPROF.so python tools/prof_hhqr.py m n
"""
import ctypes
import os
import sys
from collections import defaultdict

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
import paper_1401_5171_b200 as oqr  # noqa: E402

NAMES = {2: "copy Z->X", 3: "column partials", 4: "column barrier+reads", 5: "column update",
         6: "panel V^T[V C] partials", 7: "panel reduce-scatter (2 barriers)", 9: "panel T + trailing update",
         10: "Y: V^T Y partials", 11: "Y: reduce-scatter (2 barriers)", 12: "Y: update", 13: "tail"}


def main():
    m, n = int(sys.argv[1]), int(sys.argv[2])
    p = gen.problem(m, n, 1.0, 1e2, 5, with_A=False)
    Z = torch.from_numpy(p.Z).cuda()
    L = oqr.lib()
    f = L.oqr_exp_hh_prof
    f.restype = ctypes.c_int
    f.argtypes = [ctypes.c_void_p, ctypes.c_int]
    buf = (ctypes.c_ulonglong * 16384)()
    for rep in range(3):
        f(buf, 16384)
        oqr.hhqr(Z, m=m)
        torch.cuda.synchronize()
        k = f(buf, 16384)
    ev = [(int(buf[i]) >> 56, int(buf[i]) & ((1 << 56) - 1)) for i in range(k)]
    acc = defaultdict(float)
    cnt = defaultdict(int)
    for (t0, a), (t1, b) in zip(ev, ev[1:]):
        acc[t1] += (b - a) / 1e3
        cnt[t1] += 1
    tot = (ev[-1][1] - ev[0][1]) / 1e3
    print(f"hhqr m={m} n={n}: CTA 0 wall {tot:.1f} us")
    for t in sorted(acc):
        print(f"  {NAMES.get(t, t):38s} {acc[t]:9.1f} us  ({cnt[t]} x {acc[t] / cnt[t]:.2f} us)")


if __name__ == "__main__":
    main()
