"""Asynchronous, CUDA-graph-capturable entry points (oqr_*_async with a caller workspace and a
device status word): bitwise the same results as the synchronous calls, breakdown codes delivered
through d_status, and a captured CUDA graph replayed on fresh inputs."""
import pytest

import gen

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
DEV = "cuda:0"


@pytest.fixture(scope="module")
def oqr():
    import paper_1401_5171_b200 as m
    m.lib()
    return m


def buffers(oqr, m, n):
    ws = torch.empty(oqr.workspace_bytes(m, n) // 8 + 32, dtype=torch.float64, device=DEV)
    Q = torch.empty((n, m), dtype=torch.float64, device=DEV)
    R = torch.empty((n, n), dtype=torch.float64, device=DEV)
    st = torch.full((1,), -7, dtype=torch.int32, device=DEV)
    return ws, Q, R, st


@pytest.mark.parametrize("variant", ["normal", "normal2", "prequr", "prequr_stable"])
@pytest.mark.parametrize("mn", [(200, 10), (1000, 100), (333, 21)])
def test_async_equals_sync(oqr, variant, mn):
    m, n = mn
    p = gen.problem(m, n, 1e3, 1e2, 71, lda=m + (m & 1))
    A, Z = torch.from_numpy(p.A).to(DEV), torch.from_numpy(p.Z).to(DEV)
    Qs, Rs, ss = oqr.VARIANTS[variant](A, Z)
    for use_ws in (True, False):
        ws, Q, R, st = buffers(oqr, m, n)
        oqr.VARIANTS_ASYNC[variant](A, Z, Q, R, ws if use_ws else None, st)
        torch.cuda.synchronize()
        assert int(st.item()) == ss == 0
        assert torch.equal(Q, Qs) and torch.equal(R, Rs)


def test_async_breakdown_status(oqr):
    p = gen.problem(400, 20, 1e8, 1e6, 77, ucase="split")     # kappa(G) = 1e20
    A, Z = torch.from_numpy(p.A).to(DEV), torch.from_numpy(p.Z).to(DEV)
    ws, Q, R, st = buffers(oqr, 400, 20)
    oqr.normal_async(A, Z, Q, R, ws, st)
    torch.cuda.synchronize()
    _, _, ss = oqr.normal(A, Z)
    assert int(st.item()) == ss and 1 <= ss <= 20


def test_workspace_too_small_is_rejected(oqr):
    p = gen.problem(200, 10, 1e2, 1e2, 1)
    A, Z = torch.from_numpy(p.A).to(DEV), torch.from_numpy(p.Z).to(DEV)
    _, Q, R, st = buffers(oqr, 200, 10)
    small = torch.empty(16, dtype=torch.float64, device=DEV)
    with pytest.raises(oqr.OqrError) as e:
        oqr.normal_async(A, Z, Q, R, small, st)
    assert e.value.status == -102


@pytest.mark.parametrize("variant", ["normal", "prequr"])
def test_cuda_graph_capture_and_replay(oqr, variant):
    m, n = 4000, 50
    p = gen.problem(m, n, 1e4, 1e3, 72)
    A = torch.from_numpy(p.A).to(DEV)
    Zin = torch.from_numpy(p.Z).to(DEV)
    ws, Q, R, st = buffers(oqr, m, n)
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):                       # warm-up outside capture (lazy init)
        oqr.VARIANTS_ASYNC[variant](A, Zin, Q, R, ws, st)
    torch.cuda.current_stream().wait_stream(side)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        oqr.VARIANTS_ASYNC[variant](A, Zin, Q, R, ws, st)
    for seed in (73, 74, 75):
        q = gen.problem(m, n, 1e4, 1e3, seed, with_A=False)
        Zin.copy_(torch.from_numpy(q.Z))
        g.replay()
        torch.cuda.synchronize()
        Qs, Rs, ss = oqr.VARIANTS[variant](A, Zin)
        assert int(st.item()) == ss == 0
        assert torch.equal(R, Rs) and torch.equal(Q, Qs)
