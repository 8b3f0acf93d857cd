"""Pins of the oracle's univariate layer (oracle/splines.py) against closed forms.

Each pin is independent of the code it checks: Bernstein-polynomial integrals, classical Gauss
rules, finite differences, and the commuting-diagram identity of 1D integration by parts.
"""
from math import comb

import numpy as np
import pytest

from oracle import splines as S


def test_knot_examples():
    # S:L55-57 (make_open_knot_vector examples)
    assert np.allclose(S.open_knots(2, 2), [0, 0, 0, 0.5, 1, 1, 1])
    assert len(S.open_knots(4, 8)) - 4 - 1 == 12
    assert np.allclose(S.derived_knots(S.open_knots(2, 2)), [0, 0, 0.5, 1, 1])
    # dims a = n+p-2 (trimmed S_p and S_{p-2}(Xi'')), b = n+p-1 (P:L173 squareness)
    for p in (2, 3, 4):
        for n in (1, 3, 8):
            assert S.space_dim("Sp", p, n) == S.space_dim("Dp2", p, n) == n + p - 2
            assert S.space_dim("Sp1", p, n) == S.space_dim("Dp1", p, n) == n + p - 1


def test_gauss_rule_classical():
    x, w = S.gauss_rule(1, 1)
    assert np.allclose(x, [0.5]) and np.allclose(w, [1.0])
    x, w = S.gauss_rule(1, 2)
    assert np.allclose(np.sort(x), [0.5 - 0.5 / np.sqrt(3), 0.5 + 0.5 / np.sqrt(3)], atol=1e-15)
    x, w = S.gauss_rule(4, 3)
    assert abs(np.sum(w * x ** 5) - 1 / 6) < 1e-15


@pytest.mark.parametrize("p", [2, 3, 4])
@pytest.mark.parametrize("n", [1, 2, 5])
def test_partition_of_unity_and_cs_integral(p, n):
    x = np.random.default_rng(1).uniform(0, 1, 100)
    X = S.open_knots(p, n)
    for q, K in ((p, X), (p - 1, S.derived_knots(X))):
        assert np.abs(S.bspline_values(K, q, x).sum(1) - 1).max() < 1e-14
    # int CS = 1 for both CS spaces (reading Z2)
    xq, wq = S.gauss_rule(n, p + 1)
    for sp in ("Sp1", "Dp2"):
        ints = wq @ S.space_values(sp, p, n, xq)
        assert np.abs(ints - 1).max() < 1e-14


def _bern(m, i, k, j):
    """int_0^1 b_i^m b_j^k dx = C(m,i) C(k,j) / ((m+k+1) C(m+k, i+j))  (closed form)."""
    return comb(m, i) * comb(k, j) / ((m + k + 1) * comb(m + k, i + j))


@pytest.mark.parametrize("p", [2, 3, 4])
def test_one_element_bernstein_closed_forms(p):
    """At n = 1 every space is a Bernstein basis: S_p trimmed = b^p_1..b^p_{p-1}; CS of degree q
    on [0,1] = (q+1) b^q_i.  Hat{G} = int D'' B, Hat{M} = int B' D'."""
    n = 1
    G = S.gram_1d("Dp2", "Sp", p, n)
    Mh = S.gram_1d("Dp1", "Sp1", p, n)
    Gex = np.array([[(p - 1) * _bern(p - 2, k, p, c + 1) for c in range(p - 1)] for k in range(p - 1)])
    Mex = np.array([[p * _bern(p - 1, j, p - 1, k) for k in range(p)] for j in range(p)])
    assert np.abs(G - Gex).max() < 1e-15
    assert np.abs(Mh - Mex).max() < 1e-15
    GBp = S.gram_1d("Sp", "Sp", p, n)
    assert np.abs(GBp - np.array([[_bern(p, i + 1, p, j + 1) for j in range(p - 1)]
                                  for i in range(p - 1)])).max() < 1e-15
    if p == 2:
        # SURVEY A1 / reading Z1: Hat{G} = [1/3] (not SPEC's 2/3); Gamma_B^2 = 2/15
        assert abs(G[0, 0] - 1 / 3) < 4e-16
        assert np.abs(Mh - np.array([[2 / 3, 1 / 3], [1 / 3, 2 / 3]])).max() < 4e-16
        assert abs(GBp[0, 0] - 2 / 15) < 4e-16


def _d_primal(a):
    """(b x a) primal derivative on trimmed coefficients: (du)_j = u_j - u_{j-1}."""
    D = np.zeros((a + 1, a))
    for j in range(a + 1):
        if j < a:
            D[j, j] = 1
        if j >= 1:
            D[j, j - 1] = -1
    return D


@pytest.mark.parametrize("p", [2, 3, 4])
@pytest.mark.parametrize("n", [1, 2, 7, 32])
def test_commuting_diagram_and_bands(p, n):
    """1D integration by parts with the trimmed primal space: Hat{M} d = d Hat{G};
    column sums of Hat{M} are 1 (int D' = 1, sum B' = 1); half-bandwidth p-1 (D2)."""
    G = S.gram_1d("Dp2", "Sp", p, n)
    Mh = S.gram_1d("Dp1", "Sp1", p, n)
    a = n + p - 2
    D = _d_primal(a)
    assert np.abs(Mh @ D - D @ G).max() < 5e-15
    assert np.abs(Mh.sum(0) - 1).max() < 5e-15
    for A in (G, Mh):
        i, j = np.nonzero(np.abs(A) > 1e-15)
        assert np.max(np.abs(i - j), initial=0) <= p - 1


@pytest.mark.parametrize("p", [2, 3, 4])
def test_derivative_identity_finite_differences(p):
    """f = sum c_i B_i (S_p, untrimmed) has f' = sum (c_{j+1} - c_j) D'_j in the CS basis of
    S_{p-1}(Xi') -- checked against central finite differences."""
    n = 5
    X = S.open_knots(p, n)
    c = np.random.default_rng(2).standard_normal(n + p)
    x = np.random.default_rng(3).uniform(0.01, 0.99, 50)
    hh = 1e-6
    fd = (S.bspline_values(X, p, x + hh) @ c - S.bspline_values(X, p, x - hh) @ c) / (2 * hh)
    X1 = S.derived_knots(X)
    Dcs = S.bspline_values(X1, p - 1, x) * S.cs_scale(X1, p - 1)[None, :]
    assert np.abs(Dcs @ np.diff(c) - fd).max() < 1e-6 * (1 + np.abs(fd).max())
    # and the oracle's own derivative routine agrees
    assert np.abs(S.bspline_derivatives(X, p, x) @ c - fd).max() < 1e-6 * (1 + np.abs(fd).max())
