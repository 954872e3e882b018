"""Per-call time of oqr_normal (synchronous) vs the same step replayed as a captured CUDA graph
(oqr_normal_async + caller workspace), for the small configs where launch/sync latency matters.
    python tools/time_graph.py [config ...]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import gen  # noqa: E402
import paper_1401_5171_b200 as oqr  # noqa: E402

for cfg in [int(c) for c in (sys.argv[1:] or ["0", "1", "4"])]:
    p = gen.config(cfg)
    m, n = p.m, p.n
    A, Z = torch.from_numpy(p.A).cuda(), torch.from_numpy(p.Z).cuda()
    Q = torch.empty((n, m), dtype=torch.float64, device="cuda")
    R = torch.empty((n, n), dtype=torch.float64, device="cuda")
    ws = torch.empty(oqr.workspace_bytes(m, n) // 8 + 32, dtype=torch.float64, device="cuda")
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    reps = 200 if m <= 4000 else 20
    for _ in range(3):
        oqr.normal(A, Z, Q, R)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        oqr.normal(A, Z, Q, R)
    t_sync = (time.perf_counter() - t) / reps
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        oqr.normal_async(A, Z, Q, R, ws, st)
    torch.cuda.current_stream().wait_stream(side)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        oqr.normal_async(A, Z, Q, R, ws, st)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    t_graph = e0.elapsed_time(e1) / reps * 1e-3
    fl = 2.0 * m * m * n + 2.0 * m * n * n
    print(f"config {cfg} m={m} n={n}: oqr_normal (sync, wall) {t_sync * 1e3:.4f} ms = {fl / t_sync / 1e12:.2f} TF/s; "
          f"graph replay {t_graph * 1e3:.4f} ms = {fl / t_graph / 1e12:.2f} TF/s; status {int(st.item())}")
