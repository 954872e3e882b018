"""Time K6 (Householder QR, oqr_hhqr) and oqr_prequr_hh against oqr_prequr / oqr_prequr_stable.

    python tools/time_hhqr.py [m n ...]
"""
import sys
import time

import torch

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import gen  # noqa: E402
import paper_1401_5171_b200 as oqr  # noqa: E402


def t_events(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    return min(ts), sorted(ts)[len(ts) // 2]


def main():
    shapes = [(int(a), int(b)) for a, b in zip(sys.argv[1::2], sys.argv[2::2])] or \
        [(4000, 50), (10000, 100), (20000, 100), (40000, 200), (100000, 200)]
    for m, n in shapes:
        p = gen.problem(m, n, 1.0, 1e2, 5, with_A=False)
        Z = torch.from_numpy(p.Z).cuda()
        oqr.timing_enable(True)
        oqr.timing_reset()
        oqr.hhqr(Z, m=m)
        torch.cuda.synchronize()
        k6 = oqr.timing_read_kernel("K6")[0]
        oqr.timing_enable(False)
        mn, md = t_events(lambda: oqr.hhqr(Z, m=m))
        fl = 4.0 * m * n * n - 4.0 * n ** 3 / 3   # geqrf 2mn^2 - 2n^3/3 + orgqr 2mn^2 - 2n^3/3
        print(f"hhqr m={m} n={n}: min {mn:.3f} ms, median {md:.3f} ms (K6 event {k6:.3f} ms), "
              f"{fl / (mn * 1e-3) / 1e9:.1f} GFLOP/s", flush=True)


if __name__ == "__main__":
    main()
