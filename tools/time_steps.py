"""Per-step CUDA-event timings through the step exports (pack+K1+K1r, K2, K3) and the three
variants, for one BASELINE config (or "m,n").      python tools/time_steps.py [config|m,n] [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import gen  # noqa: E402
import paper_1401_5171_b200 as oqr  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
if cfg in gen.TRIDIAG_CONFIGS:
    d, e, p = gen.tridiag_config(cfg)
    m, n = p.m, p.n
    dg, eg = torch.from_numpy(d).cuda(), torch.from_numpy(e).cuda()
    Z = torch.from_numpy(p.Z).cuda()

    def timed(fn):
        fn()
        fn()  # a second identical synchronous call is captured into the library's cached graph
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    G = oqr.gram_tridiag(dg, eg, Z)
    R, info = oqr.potrf(G)
    res = {"gram_tridiag (K4t fused stencil, K1r)": timed(lambda: oqr.gram_tridiag(dg, eg, Z, G)),
           "potrf (K2)": timed(lambda: oqr.potrf(G, R, info)), "trsm (K3)": timed(lambda: oqr.trsm(Z, R))}
    for v in ("normal", "normal2", "prequr", "prequr_hh"):
        res[v] = timed(lambda: oqr.VARIANTS_TRIDIAG[v](dg, eg, Z))
    fl = 2.0 * m * n * n
    print(f"tridiag config {cfg} m={m} n={n}: " + ", ".join(f"{k} {v:.4f} ms" for k, v in res.items()) +
          f"; normal {fl / res['normal'] / 1e9:.2f} TFLOP/s (2mn^2 normalisation)")
    sys.exit(0)
if "," in cfg:                       # "m,n": a synthetic problem off the BASELINE list
    mm, nn = (int(x) for x in cfg.split(","))
    p = gen.problem(mm, nn, 1e3, 1e2, 7)
else:
    p = gen.config(int(cfg))
m, n = p.m, p.n
A = torch.from_numpy(p.A).cuda()
Z = torch.from_numpy(p.Z).cuda()


def timed(fn):
    fn()
    fn()  # a second identical synchronous call is captured into the library's cached graph
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


G = oqr.gram(A, Z)
R, info = oqr.potrf(G)
torch.cuda.synchronize()
assert int(info.item()) == 0
oqr.timing_enable(True)
oqr.timing_reset()
res = {"gram (pack+K1+K1r)": timed(lambda: oqr.gram(A, Z, G)),
       "K1 alone": (lambda t: t[0] / t[1])(oqr.timing_read()),
       "gram_euclid (pack+K4+K1r)": timed(lambda: oqr.gram_euclid(Z, m=m)),
       "potrf (K2)": timed(lambda: oqr.potrf(G, R, info)),
       "trsm (K3)": timed(lambda: oqr.trsm(Z, R))}
res["hhqr (K6)"] = timed(lambda: oqr.hhqr(Z, m=m))
# the variants as a user calls them: hook off (with it on the library takes neither its cached
# graphs nor the overlapped K2 -> K3 pair)
oqr.timing_enable(False)
for v in ("normal", "normal2", "prequr", "prequr_stable", "prequr_hh"):
    Q = torch.empty((n, m), dtype=torch.float64, device="cuda")
    Rv = torch.empty((n, n), dtype=torch.float64, device="cuda")
    res[v] = timed(lambda: oqr.VARIANTS[v](A, Z, Q, Rv))
fl = 2.0 * m * m * n + 2.0 * m * n * n
print(f"config {cfg} m={m} n={n}: " + ", ".join(f"{k} {v:.4f} ms" for k, v in res.items()) +
      f"; normal {fl / res['normal'] / 1e9:.1f} TFLOP/s")
