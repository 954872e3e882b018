"""include/oqr.h promises that concurrent calls on different streams are safe (stream-ordered
workspace from a mutex-guarded library pool, per-(kernel, device) attribute setup, no shared
scratch).  Four host threads (ctypes releases the GIL) each run all variants on their own stream;
every result must be bitwise the single-threaded one."""
import threading

import pytest

import gen

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def test_threads_on_separate_streams_bitwise():
    import paper_1401_5171_b200 as oqr
    probs = [gen.problem(m, n, 1e3, 1e2, 90 + i) for i, (m, n) in enumerate([(1000, 40), (2000, 100), (517, 240), (4000, 50)])]
    dev = [(torch.from_numpy(p.A).cuda(), torch.from_numpy(p.Z).cuda()) for p in probs]
    ref = {(i, v): oqr.VARIANTS[v](A, Z)[:2] for i, (A, Z) in enumerate(dev) for v in oqr.VARIANTS}
    torch.cuda.synchronize()
    results, errors = {}, []

    def worker(i):
        try:
            s = torch.cuda.Stream()
            A, Z = dev[i]
            with torch.cuda.stream(s):
                for rep in range(3):
                    for v, fn in oqr.VARIANTS.items():
                        Q, R, st = fn(A, Z, stream=s)
                        assert st == 0
                        results[(i, v, rep)] = (Q, R)
            s.synchronize()
        except Exception as e:  # pragma: no cover
            errors.append(repr(e))

    th = [threading.Thread(target=worker, args=(i,)) for i in range(len(dev))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    torch.cuda.synchronize()
    assert not errors, errors
    for (i, v, rep), (Q, R) in results.items():
        Qr, Rr = ref[(i, v)]
        assert torch.equal(Q, Qr) and torch.equal(R, Rr), (i, v, rep)


def test_pool_releases_host_call_staging():
    """oqr_normal_host streams A through a bounded ring of device chunk buffers from the library
    pool (~1 GiB, not a device copy of A): after a call on a 4.6 GB A the pool holds less than A
    (no A-sized reservation outlives the call), and oqr_pool_trim(0) empties it."""
    import numpy as np
    import paper_1401_5171_b200 as oqr
    m, n = 24000, 16                       # A = 4.6 GB > 4 GiB
    A = torch.empty((m, m), dtype=torch.float64)
    A.fill_(0.0)
    A.view(-1)[:: m + 1] = 2.0             # 2 I: SPD, trivially factorable
    Z = torch.from_numpy(np.ascontiguousarray(np.eye(m, n).T))
    Q, R, st = oqr.normal_host(A, Z)
    assert st == 0
    assert torch.allclose(R, 2.0 ** 0.5 * torch.eye(n, dtype=torch.float64))
    assert oqr.pool_reserved() < m * m * 8
    oqr.pool_trim(0)
    assert oqr.pool_reserved() == 0


@pytest.mark.parametrize("variant", ["normal", "normal2", "prequr", "prequr_stable", "prequr_hh"])
def test_cached_graph_calls_bitwise_direct(variant):
    """The second identical synchronous call of a small problem is captured into a CUDA graph and
    replayed from then on (include/oqr.h): the same kernels, so the results are bitwise the first
    (direct) call's, also for a later call with different output buffers (a new key: direct again)."""
    import paper_1401_5171_b200 as oqr
    p = gen.problem(3000, 48, 1e4, 1e3, 95)
    A, Z = torch.from_numpy(p.A).cuda(), torch.from_numpy(p.Z).cuda()
    Q = torch.empty((48, 3000), dtype=torch.float64, device="cuda")
    R = torch.empty((48, 48), dtype=torch.float64, device="cuda")
    fn = oqr.VARIANTS[variant]
    outs = []
    for _ in range(4):                     # direct, capture + replay, replay, replay
        Q.fill_(float("nan"))
        R.fill_(float("nan"))
        _, _, st = fn(A, Z, Q, R)
        assert st == 0
        outs.append((Q.clone(), R.clone()))
    for Qx, Rx in outs[1:]:
        assert torch.equal(Qx, outs[0][0]) and torch.equal(Rx, outs[0][1])
    Q2, R2, st = fn(A, Z)                  # fresh outputs: another key
    assert st == 0 and torch.equal(Q2, outs[0][0]) and torch.equal(R2, outs[0][1])


@pytest.mark.parametrize("variant", ["normal", "normal2", "prequr"])
def test_cached_graph_calls_bitwise_direct_tridiag(variant):
    """The tridiagonal family takes the cached graph too (m n^2 small): replays are bitwise the
    direct call's; a breakdown status comes back through the graph as through the direct path."""
    import paper_1401_5171_b200 as oqr
    m, n = 20000, 64
    d, e = gen.tridiag(m, 1e3)
    p = gen.problem(m, n, 1e3, 1e2, 96, with_A=False)
    dg, eg, Z = torch.from_numpy(d).cuda(), torch.from_numpy(e).cuda(), torch.from_numpy(p.Z).cuda()
    Q = torch.empty((n, m), dtype=torch.float64, device="cuda")
    R = torch.empty((n, n), dtype=torch.float64, device="cuda")
    fn = oqr.VARIANTS_TRIDIAG[variant]
    outs = []
    for _ in range(4):                     # direct, capture + replay, replay, replay
        Q.fill_(float("nan"))
        R.fill_(float("nan"))
        _, _, st = fn(dg, eg, Z, Q, R)
        assert st == 0
        outs.append((Q.clone(), R.clone()))
    for Qx, Rx in outs[1:]:
        assert torch.equal(Qx, outs[0][0]) and torch.equal(Rx, outs[0][1])
    # same pointers, new contents: a zero column of Z makes the Gram's pivot exactly 0 -- a
    # breakdown at that column, reported through the replayed graph's status word
    Z[1].zero_()
    _, _, st = fn(dg, eg, Z, Q, R)
    assert st == 2


@pytest.mark.parametrize("mn", [(3000, 48), (2500, 200), (1031, 9), (900, 232), (900, 240)])
@pytest.mark.parametrize("variant", ["normal", "normal2", "prequr", "prequr_stable", "prequr_hh"])
def test_overlapped_potrf_trsm_bitwise_serial(variant, mn):
    """K3 is launched as a programmatic dependent of K2 and follows K2's progress word block row by
    block row (session 4).  With the timing hook on the library takes the serial pair
    (K2, then K3 on the finished image): the results must be bitwise the same -- for the direct call
    and for the graph replays, where the two kernels really run concurrently.  n = 240 has no
    diagonal tiles in the image and always takes the serial pair."""
    import paper_1401_5171_b200 as oqr
    m, n = mn
    p = gen.problem(m, n, 1e3, 1e2, 97)
    A, Z = torch.from_numpy(p.A).cuda(), torch.from_numpy(p.Z).cuda()
    fn = oqr.VARIANTS[variant]
    oqr.timing_enable(True)
    try:
        Qs, Rs, st = fn(A, Z)
    finally:
        oqr.timing_enable(False)
    assert st == 0
    Q = torch.empty((n, m), dtype=torch.float64, device="cuda")
    R = torch.empty((n, n), dtype=torch.float64, device="cuda")
    for rep in range(4):                   # direct, capture + replay, replay, replay
        Q.fill_(float("nan"))
        R.fill_(float("nan"))
        _, _, st = fn(A, Z, Q, R)
        assert st == 0
        assert torch.equal(Q, Qs) and torch.equal(R, Rs), (variant, mn, rep)


@pytest.mark.parametrize("variant", ["normal", "normal2", "prequr"])
def test_overlapped_potrf_trsm_breakdown(variant):
    """A breakdown inside the overlapped pair: K2 tells K3 to stop through the progress word, the
    status is the serial pair's, and the next (healthy) call through the same cached graph is
    bitwise the serial result again."""
    import paper_1401_5171_b200 as oqr
    m, n = 3000, 120
    p = gen.problem(m, n, 1e2, 1e2, 98)
    A, Z = torch.from_numpy(p.A).cuda(), torch.from_numpy(p.Z).cuda()
    fn = oqr.VARIANTS[variant]
    oqr.timing_enable(True)
    try:
        Qs, Rs, st = fn(A, Z)
        assert st == 0
        Zb = Z.clone()
        Zb[77].zero_()                     # column 77 of Z is zero: pivot 78 of the first Cholesky is 0
        _, _, stb = fn(A, Zb, check=False)
    finally:
        oqr.timing_enable(False)
    assert stb == 78
    Q = torch.empty((n, m), dtype=torch.float64, device="cuda")
    R = torch.empty((n, n), dtype=torch.float64, device="cuda")
    Zw = Z.clone()
    for rep in range(6):                   # healthy / broken alternate through the same pointers
        broken = rep % 2 == 1
        Zw.copy_(Zb if broken else Z)
        _, _, st = fn(A, Zw, Q, R, check=False)
        if broken:
            assert st == 78, (variant, rep, st)
        else:
            assert st == 0 and torch.equal(Q, Qs) and torch.equal(R, Rs), (variant, rep)
