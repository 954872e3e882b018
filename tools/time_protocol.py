"""SURVEY s8(d) timing protocol for every BASELINE config: L2 flushed before each repetition
(a write of 2x the 126 MB L2), 2 warm-ups, 10 repetitions, min (the paper's "minimum of 10",
PAPER.md:962) and median.  T_call = host wall time around the synchronous C-ABI call
(oqr_normal / oqr_normal2 / oqr_prequr); T_S1 = CUDA events around the asynchronous oqr_gram
(pack + K1 + K1r) on the current stream.  GFLOP/s: T_call with the paper's 2m^2n + 2mn^2,
T_S1 with 2m^2n.

    python tools/time_protocol.py [configs, e.g. 0,1,2,3,4] [reps]
"""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import gen  # noqa: E402
import paper_1401_5171_b200 as oqr  # noqa: E402

cfgs = [int(c) for c in (sys.argv[1] if len(sys.argv) > 1 else "0,1,2,3,4").split(",")]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
flush_buf = torch.empty(2 * 126 * 2 ** 20 // 8, dtype=torch.float64, device="cuda")


def flush():
    flush_buf.fill_(1.0)
    torch.cuda.synchronize()


def stats(ts):
    return min(ts), statistics.median(ts)


print(f"# L2 flushed (256 MB write) before every repetition; 2 warm-ups, {reps} repetitions; min / median")
for c in cfgs:
    p = gen.config(c)
    m, n = p.m, p.n
    A = torch.from_numpy(p.A).cuda()
    Z = torch.from_numpy(p.Z).cuda()
    Q = torch.empty((n, m), dtype=torch.float64, device="cuda")
    R = torch.empty((n, n), dtype=torch.float64, device="cuda")
    G = torch.empty((n, n), dtype=torch.float64, device="cuda")
    fl_call = 2.0 * m * m * n + 2.0 * m * n * n
    fl_s1 = 2.0 * m * m * n
    out = []
    ts = []
    for i in range(reps + 2):
        flush()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        oqr.gram(A, Z, G)
        e1.record()
        torch.cuda.synchronize()
        if i >= 2:
            ts.append(e0.elapsed_time(e1) * 1e-3)
    mn_, md = stats(ts)
    out.append(f"T_S1 {mn_ * 1e3:.4f} / {md * 1e3:.4f} ms = {fl_s1 / mn_ / 1e9:.0f} GFLOP/s")
    for v in ("normal", "normal2", "prequr"):
        ts = []
        for i in range(reps + 2):
            flush()
            t0 = time.perf_counter()
            _, _, st = oqr.VARIANTS[v](A, Z, Q, R)
            t1 = time.perf_counter()
            assert st == 0, (c, v, st)
            if i >= 2:
                ts.append(t1 - t0)
        mn_, md = stats(ts)
        out.append(f"{v} {mn_ * 1e3:.4f} / {md * 1e3:.4f} ms = {fl_call / mn_ / 1e9:.0f} GFLOP/s")
    print(f"config {c} m={m} n={n}: " + "; ".join(out), flush=True)
    del A, Z, Q, R, G
    torch.cuda.empty_cache()
