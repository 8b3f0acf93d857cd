"""Tier A assembly by 3D quadrature with explicit pull-backs (TEST INFRASTRUCTURE ONLY).

* Geometry F: (0,1)^3 -> Omega is a spline in S_p(Xi)^3 given by control points
  ``ctrl[(nz+p)][(ny+p)][(nx+p)][3]`` (untrimmed B-splines); ``None`` is the identity.
* Quadrature: (Q = p+1)-point Gauss per axis per element (reading Z13); the global quadrature
  grid is ordered [z-point][y-point][x-point], each axis point index = element*Q + q.
* Pull-backs (vector proxies): a 1-form with parametric proxy w^ has physical proxy
  DF^{-T} w^; a 2-form with parametric proxy w^ has physical proxy DF w^ / det DF.
* Pairings are integrals of wedge products: for the (2-form, 1-form) pairs of K1
  and K~1 the integrand is the dot product of the physical proxies, integrated over Omega.
* Masses: (eta, omega)_{L^2_gamma Lambda^2} = int_Omega gamma eta . omega dx with
  the physical 2-form proxies.

Materials and all per-quadrature-point inputs use the C-ABI layout, element-major
[ez][ey][ex][qz][qy][qx]; ``qp_elem_to_grid`` converts to the global grid order.
"""
import numpy as np
import scipy.sparse as sp

from .splines import open_knots, bspline_values, bspline_derivatives, gauss_rule, space_values
from .forms import component_spaces, component_shapes, _n3


def qp_elem_to_grid(arr, n, Q):
    """[ez][ey][ex][qz][qy][qx] (flat) -> global grid [ez*Q+qz][ey*Q+qy][ex*Q+qx] (flat)."""
    nx, ny, nz = _n3(n)
    a = np.asarray(arr).reshape(nz, ny, nx, Q, Q, Q)
    return a.transpose(0, 3, 1, 4, 2, 5).reshape(-1)


def qp_grid_to_elem(arr, n, Q):
    nx, ny, nz = _n3(n)
    a = np.asarray(arr).reshape(nz, Q, ny, Q, nx, Q)
    return a.transpose(0, 2, 4, 1, 3, 5).reshape(-1)


class Quad:
    """1D Gauss data per axis and the 3D tensor weights on the global grid."""

    def __init__(self, p, n, Q=None):
        self.p = p
        self.n = _n3(n)
        self.Q = Q if Q is not None else p + 1
        self.x1d = []
        self.w1d = []
        for a in range(3):
            x, w = gauss_rule(self.n[a], self.Q)
            self.x1d.append(x)
            self.w1d.append(w)
        wx, wy, wz = self.w1d
        self.w = (wz[:, None, None] * wy[None, :, None] * wx[None, None, :]).ravel()
        self.nqp = self.w.size


def _kron3(Vx, Vy, Vz):
    """Tensor-product basis values at the tensor-product points: rows (qz,qy,qx), cols (iz,iy,ix)."""
    return sp.kron(sp.csr_matrix(Vz), sp.kron(sp.csr_matrix(Vy), sp.csr_matrix(Vx))).tocsr()


def basis_at_qp(quad, cplx, k, comp):
    sx, sy, sz = component_spaces(cplx, k)[comp]
    p = quad.p
    V = [space_values(s, p, quad.n[a], quad.x1d[a]) for a, s in enumerate((sx, sy, sz))]
    return _kron3(*V)


def identity_ctrl(p, n):
    """Control points reproducing F = identity: Greville abscissae (affine reproduction)."""
    n = _n3(n)
    g = []
    for a in range(3):
        X = open_knots(p, n[a])
        m = n[a] + p
        g.append(np.array([X[i + 1:i + p + 1].mean() for i in range(m)]))
    gz, gy, gx = np.meshgrid(g[2], g[1], g[0], indexing="ij")
    return np.stack([gx, gy, gz], axis=-1)


class Rational:
    """A rational (NURBS) map F = sum_i w_i P_i N_i / sum_i w_i N_i over the untrimmed S_p basis
    (F is "a (rational) spline").  P: control points
    [(nz+p)][(ny+p)][(nx+p)][3]; w: positive weights [(nz+p)][(ny+p)][(nx+p)]."""

    def __init__(self, P, w):
        self.P = np.asarray(P, dtype=np.float64)
        self.w = np.asarray(w, dtype=np.float64)


def geometry_at_qp(quad, ctrl):
    """Physical points F(x_q) [nqp,3] and Jacobians DF(x_q) [nqp,3,3] (DF[i,j] = dF_i/dx^_j).
    ``ctrl``: None (identity), control points (polynomial map) or a ``Rational``.  For a rational
    map with numerator N = sum w P B and denominator W = sum w B: F = N / W and
    dF/dx^_j = (dN/dx^_j - F dW/dx^_j) / W (quotient rule)."""
    p, n = quad.p, quad.n
    if ctrl is None:
        X = np.stack(np.meshgrid(quad.x1d[2], quad.x1d[1], quad.x1d[0], indexing="ij")[::-1], -1)
        DF = np.broadcast_to(np.eye(3), (quad.nqp, 3, 3)).copy()
        return X.reshape(-1, 3), DF
    if isinstance(ctrl, Rational):
        V, D = [], []
        for a in range(3):
            X = open_knots(p, n[a])
            V.append(bspline_values(X, p, quad.x1d[a]))
            D.append(bspline_derivatives(X, p, quad.x1d[a]))
        w = ctrl.w.reshape(-1)
        wP = ctrl.P.reshape(-1, 3) * w[:, None]
        Phi = _kron3(V[0], V[1], V[2])
        dPhi = [_kron3(D[0], V[1], V[2]), _kron3(V[0], D[1], V[2]), _kron3(V[0], V[1], D[2])]
        Wq = Phi @ w
        F = (Phi @ wP) / Wq[:, None]
        DF = np.stack([(dPhi[j] @ wP - F * (dPhi[j] @ w)[:, None]) / Wq[:, None] for j in range(3)], axis=-1)
        return F, DF
    ctrl = np.asarray(ctrl, dtype=np.float64).reshape(n[2] + p, n[1] + p, n[0] + p, 3)
    V, D = [], []
    for a in range(3):
        X = open_knots(p, n[a])
        V.append(bspline_values(X, p, quad.x1d[a]))
        D.append(bspline_derivatives(X, p, quad.x1d[a]))
    c = ctrl.reshape(-1, 3)
    Phi = _kron3(V[0], V[1], V[2])
    dPhi = [_kron3(D[0], V[1], V[2]), _kron3(V[0], D[1], V[2]), _kron3(V[0], V[1], D[2])]
    F = Phi @ c
    DF = np.stack([dPhi[j] @ c for j in range(3)], axis=-1)   # [nqp, i, j]
    return F, DF


def _blocks_to_sparse(blocks):
    return sp.bmat(blocks, format="csr")


_PAIRINGS = {
    # name: (row space, column space); entries = int row ^ col
    "K0": (("dual", 3), ("primal", 0)),
    "K1": (("dual", 2), ("primal", 1)),
    "K2": (("dual", 1), ("primal", 2)),
    "K3": (("dual", 0), ("primal", 3)),
    "Kt0": (("primal", 3), ("dual", 0)),
    "Kt1": (("primal", 2), ("dual", 1)),
    "Kt2": (("primal", 1), ("dual", 2)),
    "Kt3": (("primal", 0), ("dual", 3)),
}


def pairing(quad, which, ctrl=None, physical=False):
    """Pairing matrix as a sparse block matrix.  K_k has rows = dual (3-k)-forms
    and columns = primal k-forms with eta~^T K_k w = int eta~ ^ w; K~_{3-k} has rows = primal
    k-forms and columns = dual (3-k)-forms with w^T K~_{3-k} eta~ = int w ^ eta~.

    In proxy components every wedge of a k-form with a (3-k)-form in 3D is sum_c row_c col_c
    dx^dy^dz with a + sign (dy^dz^dx = dz^dx^dy = dx^dy^dz), so the blocks are diagonal.

    physical=False: parametric proxies (the pull-back commutes with the wedge).
    physical=True (k = 1, 2 pairs only): push the 2-form and the 1-form forward with F and
    integrate the physical dot product times det DF -- pins metric independence.
    """
    rows, cols = _PAIRINGS[which]
    nc = len(component_spaces(*rows))
    R = [basis_at_qp(quad, *rows, c) for c in range(nc)]
    C = [basis_at_qp(quad, *cols, c) for c in range(nc)]
    if not physical:
        blocks = [[None] * nc for _ in range(nc)]
        for c in range(nc):
            blocks[c][c] = R[c].T @ sp.diags(quad.w) @ C[c]
        for c in range(nc):
            for c2 in range(nc):
                if blocks[c][c2] is None:
                    blocks[c][c2] = sp.csr_matrix((R[c].shape[1], C[c2].shape[1]))
        return _blocks_to_sparse(blocks)
    if which not in ("K1", "Kt1"):
        raise ValueError("physical assembly implemented for the (2-form, 1-form) pairings")
    if which == "Kt1":
        return pairing_physical_swap(quad, R, C, ctrl)
    _, DF = geometry_at_qp(quad, ctrl)
    det = np.linalg.det(DF)
    DFinvT = np.linalg.inv(DF).transpose(0, 2, 1)
    # 2-form proxy of component c basis: DF[:, :, c] * phi / det ; 1-form proxy: DFinvT[:, :, c] * psi
    blocks = [[None] * 3 for _ in range(3)]
    for c in range(3):
        for c2 in range(3):
            coef = np.einsum("qi,qi->q", DF[:, :, c] / det[:, None], DFinvT[:, :, c2]) * det * quad.w
            blocks[c][c2] = R[c].T @ sp.diags(coef) @ C[c2]
    return _blocks_to_sparse(blocks)


def pairing_physical_swap(quad, R, C, ctrl):
    """K~1 with physical pull-backs: rows are primal 2-forms (proxy DF w^/det), columns dual
    1-forms (proxy DF^{-T} w^)."""
    _, DF = geometry_at_qp(quad, ctrl)
    det = np.linalg.det(DF)
    DFinvT = np.linalg.inv(DF).transpose(0, 2, 1)
    blocks = [[None] * 3 for _ in range(3)]
    for c in range(3):
        for c2 in range(3):
            coef = np.einsum("qi,qi->q", DF[:, :, c] / det[:, None], DFinvT[:, :, c2]) * det * quad.w
            blocks[c][c2] = R[c].T @ sp.diags(coef) @ C[c2]
    return _blocks_to_sparse(blocks)


def mass2(quad, cplx, gamma_qp=None, ctrl=None):
    """2-form mass matrix with weight gamma (P:L360 M~2_{1/eps} for cplx='dual',
    P:L366 M2_{1/mu} for cplx='primal'):  M[i,j] = int_Omega gamma phys(phi_i) . phys(phi_j) dx.

    gamma_qp: values of gamma (= 1/eps or 1/mu) at the quadrature points, element-major layout;
    None means gamma = 1.
    """
    Phi = [basis_at_qp(quad, cplx, 2, c) for c in range(3)]
    _, DF = geometry_at_qp(quad, ctrl)
    det = np.linalg.det(DF)
    if gamma_qp is None:
        g = np.ones(quad.nqp)
    else:
        g = qp_elem_to_grid(gamma_qp, quad.n, quad.Q)
    blocks = [[None] * 3 for _ in range(3)]
    for c in range(3):
        for c2 in range(3):
            # sum_i (DF[i,c] phi / det)(DF[i,c2] phi' / det) * gamma * det * w
            coef = np.einsum("qi,qi->q", DF[:, :, c], DF[:, :, c2]) / det * g * quad.w
            blocks[c][c2] = Phi[c].T @ sp.diags(coef) @ Phi[c2]
    return _blocks_to_sparse(blocks)


def mass1(quad, cplx, gamma_qp=None, ctrl=None):
    """1-form mass matrix with weight gamma (scheme 1: M^1_eps for cplx='primal' on
    X^1_{h,0}, M~^1_mu for cplx='dual' on X~^1):  M[i,j] = int gamma phys(phi_i) . phys(phi_j) dx
    with the 1-form pull-back phys(phi) = DF^{-T} phi^, i.e. the weight DF^{-1} DF^{-T} det DF.
    gamma_qp: gamma (eps or mu) at the quadrature points, element-major; None = 1."""
    Phi = [basis_at_qp(quad, cplx, 1, c) for c in range(3)]
    _, DF = geometry_at_qp(quad, ctrl)
    det = np.linalg.det(DF)
    Dinv = np.linalg.inv(DF)
    G = np.einsum("qik,qjk->qij", Dinv, Dinv) * det[:, None, None]   # DF^{-1} DF^{-T} det
    g = np.ones(quad.nqp) if gamma_qp is None else qp_elem_to_grid(gamma_qp, quad.n, quad.Q)
    blocks = [[None] * 3 for _ in range(3)]
    for c in range(3):
        for c2 in range(3):
            blocks[c][c2] = Phi[c].T @ sp.diags(G[:, c, c2] * g * quad.w) @ Phi[c2]
    return _blocks_to_sparse(blocks)


def physical_qp(quad, ctrl=None):
    """Physical coordinates F(x_q) in element-major layout [ez][ey][ex][qz][qy][qx][3]."""
    F, _ = geometry_at_qp(quad, ctrl)
    return np.stack([qp_grid_to_elem(F[:, i], quad.n, quad.Q) for i in range(3)], -1)
