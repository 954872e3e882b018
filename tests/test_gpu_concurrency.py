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
