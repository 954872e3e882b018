"""Per-rank compute of the row-sharded path for N = 1, 2, 4, 8, timed ONE rank at
a time on one GPU (no rank waits on another): oqr_gram_rows on the rank's mr = m/N rows of A,
the fixed-order sum of N partials, K2 (redundant on every rank) and K3 on the rank's rows.  With
the measured exchange excluded (one all-gather of 8 n^2 bytes per rank), the slowest rank's time
bounds the strong-scaling step from below.

    python tools/time_shard.py [config] [reps]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import gen  # noqa: E402
import paper_1401_5171_b200 as oqr  # noqa: E402
from paper_1401_5171_b200.dist import row_partition  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
c = gen.CONFIGS[cfg]
m, n = c["m"], c["n"]
p = gen.config(cfg, with_A=False)
Z = torch.from_numpy(p.Z).cuda()
fl = 2.0 * m * m * n + 2.0 * m * n * n


def timed(fn):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


base = None
for N in (1, 2, 4, 8):
    parts = row_partition(m, N)
    worst = 0.0
    for r0, mr in parts[:1] + parts[-1:]:  # the first and the last shard (sizes differ by <= 64 rows)
        ldar = mr + (mr & 1)
        Ar = torch.from_numpy(gen.config_A_rows(cfg, r0, r0 + mr, lda=ldar)).cuda()
        Gp = torch.stack([oqr.gram_rows(Ar, Z, r0, mr)] * N)
        t_gram = timed(lambda: oqr.gram_rows(Ar, Z, r0, mr))
        G = oqr.sum_partials(Gp)
        t_sum = timed(lambda: oqr.sum_partials(Gp, G))
        R, info = oqr.potrf(G)
        t_potrf = timed(lambda: oqr.potrf(G, R, info))
        t_trsm = timed(lambda: oqr.trsm_rows(Z, R, r0, mr))
        worst = max(worst, t_gram + t_sum + t_potrf + t_trsm)
        del Ar
        torch.cuda.empty_cache()
    base = base or worst
    print(f"config {cfg} N={N}: per-rank compute {worst:.3f} ms (rows {parts[0][1]}..{parts[-1][1]}); "
          f"{fl / (worst * 1e-3) / 1e12:.1f} TFLOP/s whole job; efficiency vs N=1 {base / (N * worst):.3f}",
          flush=True)
