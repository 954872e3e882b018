"""Generator properties: WY closed form vs explicit reflectors,
bitwise symmetry, spectral fidelity, determinism, case selection."""
import numpy as np
import pytest

import gen


def _dense(a, rows):
    return a[:, :rows].T


def test_wy_matches_explicit_reflectors():
    p = gen.problem(60, 7, 1e3, 1e2, 11)
    Y = p.Yv.T
    H = np.eye(p.m)
    for j in range(4):
        v = Y[:, j:j + 1]
        assert abs(np.linalg.norm(v) - 1.0) < 1e-14
        H = H @ (np.eye(p.m) - 2.0 * v @ v.T)
    V = gen.wy_matrix(p.Yv, p.Tv)
    assert np.abs(H - V).max() < 1e-14


def test_A_bitwise_symmetric_and_spectrum():
    p = gen.problem(150, 9, 1e6, 1e3, 5)
    A = _dense(p.A, p.m)
    assert np.array_equal(A, A.T)
    V = gen.wy_matrix(p.Yv, p.Tv)
    assert np.abs(A - V @ np.diag(p.d) @ V.T).max() < 1e-14
    ev = np.sort(np.linalg.eigvalsh(A))[::-1]
    assert np.abs(ev - p.d).max() < 1e-13
    assert p.d[0] == 1.0 and abs(p.d[-1] * 1e6 - 1.0) < 1e-12


def test_Z_singular_values():
    p = gen.problem(120, 12, 1e2, 1e4, 7)
    sv = np.linalg.svd(_dense(p.Z, p.m), compute_uv=False)
    assert np.abs(sv - p.s).max() < 1e-13
    assert p.s[0] == 1.0 and abs(p.s[-1] * 1e4 - 1.0) < 1e-12


def test_deterministic_and_padded_ld():
    a = gen.problem(64, 5, 1e2, 1e2, 3)
    b = gen.problem(64, 5, 1e2, 1e2, 3, lda=70, ldz=66)
    assert np.array_equal(a.A, b.A[:, :64])
    assert np.array_equal(a.Z, b.Z[:, :64])
    assert np.all(np.isnan(b.A[:, 64:])) and np.all(np.isnan(b.Z[:, 64:]))   # poisoned padding
    c = gen.problem(64, 5, 1e2, 1e2, 4)
    assert not np.array_equal(a.Z, c.Z)


@pytest.mark.parametrize("ucase", ["top", "bottom", "split", "aorth"])
def test_case_columns(ucase):
    m, n = 40, 6
    p = gen.problem(m, n, 1e4, 1e2, 9, ucase=ucase)
    V = gen.wy_matrix(p.Yv, p.Tv)
    Z = _dense(p.Z, m)
    # left singular vectors of Z span the selected eigenvectors
    J = p.cols
    P = V[:, J] @ V[:, J].T
    assert np.abs(P @ Z - Z).max() < 1e-13
    if ucase == "top":
        assert list(J) == list(range(n))
    if ucase == "bottom":
        assert list(J) == list(range(m - n, m))
    if ucase in ("split", "aorth"):
        assert list(J) == [0, 1, 2, m - 3, m - 2, m - 1]
    if ucase == "aorth":
        A = _dense(p.A, m)
        assert np.abs(Z.T @ A @ Z - np.eye(n)).max() < 1e-12


def test_configs_recipe():
    p = gen.config(0)
    assert (p.m, p.n, p.kappa_a, p.kappa_z, p.seed) == (200, 10, 1e2, 1e2, 0x14015171)
    w = gen.witness(with_A=False)
    assert w.m == 10000 and w.n == 100 and w.ucase == "split"


def test_A_rows_bitwise_equal_to_full_rows():
    # the row shard of one rank (multi-GPU path) holds exactly the same bits as the full A
    p = gen.problem(333, 7, 1e4, 1e2, 19)
    full = _dense(p.A, 333)
    for r0, r1 in ((0, 64), (64, 200), (200, 333), (17, 18)):
        blk = gen.A_rows(333, 1e4, 19, r0, r1, lda=r1 - r0 + 2)
        assert np.array_equal(blk[:, : r1 - r0].T, full[r0:r1, :])


def test_input_bytes_match_the_recorded_hashes():
    """the bytes of the generated inputs are recorded (profiles/r01_input_hashes.txt,
    tools/input_hashes.py); the small ones are regenerated here and must match bit for bit."""
    import hashlib
    import os
    rec = open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                            "r01_input_hashes.txt")).read().splitlines()
    sha = lambda a: hashlib.sha256(memoryview(a).cast("B")).hexdigest()
    for k in (0, 1):
        p = gen.config(k)
        assert f"configs[{k}] m={p.m} n={p.n}  A {sha(p.A)}  Z {sha(p.Z)}" in rec
    d, e, p = gen.tridiag_config("t")
    assert f"tridiag t m={p.m} n={p.n}  d {sha(d)}  e {sha(e)}  Z {sha(p.Z)}" in rec


@pytest.mark.parametrize("ucase", ["random", "top", "bottom", "split", "aorth"])
def test_haar_construction(ucase):
    """PAPER.md:743-756 with dense random orthogonal V, W (and U, case 4): V orthogonal, A bitwise
    symmetric with eigenpairs (d, V), Z = U diag(s) W^T with orthonormal U, W."""
    m, n = 80, 10
    p = gen.problem_haar(m, n, 1e6, 1e3, 7, ucase)
    V, W = p.V, p.W
    assert np.abs(V.T @ V - np.eye(m)).max() < 1e-14
    assert np.abs(W.T @ W - np.eye(n)).max() < 1e-14
    A, Z = _dense(p.A, m), _dense(p.Z, m)
    assert np.array_equal(A, A.T)
    assert np.abs(A @ V - V * p.d).max() < 1e-14
    sv = np.linalg.svd(Z, compute_uv=False)
    assert np.abs(sv - np.sort(p.s)[::-1]).max() <= 1e-14 * p.s.max()
    if ucase == "random":
        assert list(p.cols) == [-1] * n
        # a Haar U is not aligned with any few eigenvectors: every eigen-direction carries weight
        Uz = np.linalg.svd(Z, full_matrices=False)[0]
        w = np.linalg.norm(V.T @ Uz, axis=1)
        assert w.min() > 1e-3 and w.max() < 0.9
    else:
        J = p.cols
        P = V[:, J] @ V[:, J].T
        assert np.abs(P @ Z - Z).max() < 1e-13 * np.abs(Z).max()
    if ucase == "aorth":
        assert np.abs(Z.T @ A @ Z - np.eye(n)).max() < 100 * m * 2.0 ** -53 * p.kappa_a   # u ||Z||^2 ||A||


def test_haar_deterministic_and_substreams():
    a = gen.problem_haar(40, 5, 1e3, 1e2, 3, "random")
    b = gen.problem_haar(40, 5, 1e3, 1e2, 3, "random", lda=41, ldz=43)
    assert np.array_equal(a.A, b.A[:, :40]) and np.array_equal(a.Z, b.Z[:, :40])
    assert np.all(np.isnan(b.A[:, 40:])) and np.all(np.isnan(b.Z[:, 40:]))
    c = gen.problem_haar(40, 5, 1e3, 1e2, 3, "top")
    assert np.array_equal(a.A, c.A)                 # V depends on the seed only
    assert not np.array_equal(a.Z, c.Z)
