"""Pins for the tridiagonal-A oracle (NEXT-N3).

* The tridiagonal Gram is bitwise the dense oracle's Gram of the densified T (the dense path is
  itself pinned to the paper in test_oracle_pins.py), and so are the three variants.
* Closed form: with Z = columns of T's exact eigenvectors (sin vectors) scaled by s_k, G = diag of
  s_k^2 lambda_k within the Gram error bound, and R = diag(s_k sqrt(lambda_k)) (Theorem 1).
* SPEC.md:116 worked example of the stencil: diag 2, offdiag -1, X = [1,1,1] -> [1, 0, 1].
"""
import numpy as np
import pytest

import gen
import oracle
from oracle import U


def test_spec_stencil_example():
    d, e = np.array([2.0, 2.0, 2.0]), np.array([-1.0, -1.0])
    X = oracle.to_cm(np.ones((3, 1)))
    G = oracle.gram_tridiag(d, e, X, 3)             # X^T (T X) = [1,1,1].[1,0,1] = 2
    assert G[0, 0] == 2.0


def test_kappa_of_generated_T_is_exact():
    for m, ka in ((50, 1e3), (2000, 1e5)):
        d, e = gen.tridiag(m, ka)
        lam = np.linalg.eigvalsh(oracle.from_cm(oracle.densify_tridiag(d, e), m))
        assert abs(lam[-1] / lam[0] / ka - 1.0) < 1e-8


@pytest.mark.parametrize("variant", ["normal", "normal2", "prequr"])
def test_tridiag_equals_dense_on_densified_bitwise(variant):
    m, n = 300, 11
    d, e = gen.tridiag(m, 1e4)
    p = gen.problem(m, n, 1e4, 1e2, 9, with_A=False)
    Ad = oracle.densify_tridiag(d, e)
    assert np.array_equal(oracle.gram_tridiag(d, e, p.Z, m), oracle.gram(Ad, p.Z, m))
    Qt, Rt, it = oracle.VARIANTS_TRIDIAG[variant](d, e, p.Z, m)
    Qd, Rd, idd = oracle.VARIANTS[variant](Ad, p.Z, m)
    assert it == idd == 0
    assert np.array_equal(Rt, Rd) and np.array_equal(Qt, Qd)


def test_eigenvector_closed_form():
    m, n, ka = 400, 8, 1e6
    d, e = gen.tridiag(m, ka)
    ks = [1, 2, 3, 50, 100, 200, 399, 400]
    lam, V = gen.tridiag_eigen(m, ka, ks)
    s = np.logspace(0, -3, n)
    Z = V * s
    Q, R, info = oracle.normal_tridiag(d, e, oracle.to_cm(Z), m)
    assert info == 0
    Rd = oracle.from_cm(R, n)
    expect = s * np.sqrt(lam)
    assert np.allclose(np.diag(Rd), expect, rtol=1e-9, atol=0)
    off = np.abs(Rd - np.diag(np.diag(Rd))).max()
    assert off <= 1e-9 * expect.max()
    assert oracle.orth_error_tridiag(d, e, Q, m) < 1e-9


def test_dd_orth_tridiag_matches_dense_checker():
    # the tridiagonal checker forms the same double-double sums as the dense one on the densified T
    # (the dense one only adds exact zeros), so the rounded E agrees to far below u
    m, n = 250, 9
    d, e = gen.tridiag(m, 1e5)
    p = gen.problem(m, n, 1e5, 1e3, 12, with_A=False)
    Q, _, info = oracle.normal_tridiag(d, e, p.Z, m)
    assert info == 0
    Et = oracle.orth_error_tridiag(d, e, Q, m)
    Ed = oracle.orth_error(oracle.densify_tridiag(d, e), Q, m)
    assert abs(Et - Ed) <= 1e-6 * U * max(Ed, 1e-16) + 1e-30
