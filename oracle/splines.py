"""Univariate splines for the oracle (TEST INFRASTRUCTURE ONLY, see oracle/__init__.py).

Follows PAPER.md sec. 2.3 for the p-open knot vector Xi and the derived Xi', Xi'',
and sec. 4.1 for the choice of bases:
  * primal S_p(Xi)        : B-splines, first and last removed (homogeneous BC)
  * primal S_{p-1}(Xi')   : scaled Curry--Schoenberg (CS) splines
  * dual   S_{p-1}(Xi')   : B-splines
  * dual   S_{p-2}(Xi'')  : CS splines
CS scaling (reading Z2 in DESIGN.md): D_i = (q+1)/(xi_{i+q+1}-xi_i) * B_{i,q}, so int D_i = 1.
"""
import numpy as np


def open_knots(p, n):
    """p-open uniform knot vector with n elements and simple interior knots."""
    if p < 0 or n < 1:
        raise ValueError("need p >= 0 and n >= 1")
    return np.concatenate([np.zeros(p + 1), np.arange(1, n) / n, np.ones(p + 1)])


def derived_knots(knots):
    """Xi' = Xi without its first and last knot."""
    return np.asarray(knots)[1:-1]


def bspline_values(knots, q, x):
    """Cox--de Boor recursion: returns V[len(x), m] with V[k, i] = B_{i,q}(x_k).

    Plain textbook recursion over the degree; 0/0 := 0.  The last non-empty knot span is
    closed on the right so that x = 1 is covered.
    """
    knots = np.asarray(knots, dtype=np.float64)
    x = np.atleast_1d(np.asarray(x, dtype=np.float64))
    nk = len(knots)
    # degree 0
    B = np.zeros((len(x), nk - 1))
    last = np.max(np.nonzero(knots[1:] > knots[:-1])[0])
    for i in range(nk - 1):
        if knots[i + 1] > knots[i]:
            if i == last:
                B[:, i] = (x >= knots[i]) & (x <= knots[i + 1])
            else:
                B[:, i] = (x >= knots[i]) & (x < knots[i + 1])
    for d in range(1, q + 1):
        Bn = np.zeros((len(x), nk - 1 - d))
        for i in range(nk - 1 - d):
            den1 = knots[i + d] - knots[i]
            den2 = knots[i + d + 1] - knots[i + 1]
            t = np.zeros(len(x))
            if den1 > 0:
                t += (x - knots[i]) / den1 * B[:, i]
            if den2 > 0:
                t += (knots[i + d + 1] - x) / den2 * B[:, i + 1]
            Bn[:, i] = t
        B = Bn
    return B


def bspline_derivatives(knots, q, x):
    """First derivatives of the degree-q B-splines (textbook formula
    B'_{i,q} = q/(xi_{i+q}-xi_i) B_{i,q-1} - q/(xi_{i+q+1}-xi_{i+1}) B_{i+1,q-1})."""
    knots = np.asarray(knots, dtype=np.float64)
    x = np.atleast_1d(np.asarray(x, dtype=np.float64))
    m = len(knots) - q - 1
    if q == 0:
        return np.zeros((len(x), m))
    Bl = bspline_values(knots, q - 1, x)  # m+1 functions
    D = np.zeros((len(x), m))
    for i in range(m):
        den1 = knots[i + q] - knots[i]
        den2 = knots[i + q + 1] - knots[i + 1]
        if den1 > 0:
            D[:, i] += q / den1 * Bl[:, i]
        if den2 > 0:
            D[:, i] -= q / den2 * Bl[:, i + 1]
    return D


def cs_scale(knots, q):
    """Curry--Schoenberg scale (q+1)/(xi_{i+q+1}-xi_i) of each degree-q function (reading Z2)."""
    knots = np.asarray(knots, dtype=np.float64)
    m = len(knots) - q - 1
    return np.array([(q + 1) / (knots[i + q + 1] - knots[i]) for i in range(m)])


def gauss_rule(n, Q):
    """Q-point Gauss--Legendre rule on each of the n uniform elements of [0,1] (reading Z13).

    Returns (points[n*Q], weights[n*Q]) ordered element by element.
    """
    g, w = np.polynomial.legendre.leggauss(Q)
    pts, wts = [], []
    for e in range(n):
        a, b = e / n, (e + 1) / n
        pts.append(a + (g + 1) * (b - a) / 2)
        wts.append(w * (b - a) / 2)
    return np.concatenate(pts), np.concatenate(wts)


# --- the four univariate spaces of sec. 4.1 -------------------------------------

SPACES = ("Sp", "Sp1", "Dp1", "Dp2", "SpF")
"""Sp  = primal S_p(Xi) trimmed, B-splines         (dim a = n+p-2)
   Sp1 = primal S_{p-1}(Xi') CS                     (dim b = n+p-1)
   Dp1 = dual   S_{p-1}(Xi') B-splines              (dim b)
   Dp2 = dual   S_{p-2}(Xi'') CS                    (dim a)
   SpF = primal S_p(Xi) untrimmed, B-splines       (dim a + 2: the full X^k_h of the lifting,
         P:L450-490, whose first and last functions carry the boundary values)"""


def space_dim(space, p, n):
    return {"Sp": n + p - 2, "Sp1": n + p - 1, "Dp1": n + p - 1, "Dp2": n + p - 2, "SpF": n + p}[space]


def space_values(space, p, n, x):
    """Values of the basis of one of the four univariate spaces at points x: V[len(x), dim]."""
    X = open_knots(p, n)
    X1 = derived_knots(X)
    X2 = derived_knots(X1)
    if space == "Sp":
        return bspline_values(X, p, x)[:, 1:-1]
    if space == "SpF":
        return bspline_values(X, p, x)
    if space == "Sp1":
        return bspline_values(X1, p - 1, x) * cs_scale(X1, p - 1)[None, :]
    if space == "Dp1":
        return bspline_values(X1, p - 1, x)
    if space == "Dp2":
        return bspline_values(X2, p - 2, x) * cs_scale(X2, p - 2)[None, :]
    raise ValueError(space)


def gram_1d(row_space, col_space, p, n, Q=None):
    """Dense 1D Gram/pairing matrix  G[i, j] = int_0^1 row_i(x) col_j(x) dx  by Gauss quadrature.

    Hat{G} = gram_1d('Dp2', 'Sp')  and  Hat{M} = gram_1d('Dp1', 'Sp1');
    the separable-Hodge Grams are gram_1d(s, s) for s in the four spaces.
    """
    Q = Q if Q is not None else p + 1
    x, w = gauss_rule(n, Q)
    R = space_values(row_space, p, n, x)
    C = space_values(col_space, p, n, x)
    return R.T @ (w[:, None] * C)
