"""Inhomogeneous Dirichlet data for E by lifting (sec. 3.5) and the coaxial-cable
TEM workload (sec. 5.2) -- TEST INFRASTRUCTURE ONLY.

The paper's formulation, written out literally with assembled matrices (tier A):

* E_h = E_{h,0} + E_{h,b}, E_{h,b} in X^1_h (the full primal space: untrimmed S_p, forms.py
  'primalF') with non-zero coefficients only on boundary functions, "computed through a local
  projection of the boundary conditions on its trace space";
* the second scheme's Hodge star solves (K1)_0 e_0 = M~2_{1/eps} d - (K1)_b e_b with
  K1 the pairing of X~^2 with the full X^1_h split into interior / boundary columns;
* B_h lives in X^2_h, D1 maps X^1_h -> X^2_h, and M2_{1/mu} has columns in X^2_h;
* the data are separable in space and time, E_b(x, t) = g(t) E_s(x), so e_b(t) = g(t) e^_b.

Reading Z29: the local projection is the unweighted parametric L2 projection, on each
Dirichlet face, of each tangential covariant component e^_c = DF[:, c] . E(F(x^)) onto that face's
trace space (the component's own direction S_{p-1}, the other tangential direction S_p with its end
functions removed where the adjacent face carries homogeneous data).

Coax (reading Z29): the quarter annulus 1 < r < sqrt2 (r1 = 1, r2 = sqrt2), 0 < z < 1, with the
standing TEM mode E = (1/r) sin(pi z) cos(pi t) r-hat, H = B = -(1/r) cos(pi z) sin(pi t) phi-hat
(eps = mu = 1): PEC on the cylinders and on z = 0, 1; inhomogeneous Dirichlet data E_r on the symmetry
planes theta = 0, pi/2 (the parametric faces y^ = 0, 1).
"""
import numpy as np
import scipy.sparse as sp

from . import forms
from .assemble import Quad, basis_at_qp, geometry_at_qp, mass2, pairing, qp_grid_to_elem, _blocks_to_sparse
from .scheme import TierA
from .splines import gauss_rule, gram_1d, space_values
from .structured import kron3


# ---- the exact TEM mode of the coax (Collin ch. 3) --------------------------------------

R1, R2 = 1.0, np.sqrt(2.0)


def tem_E(X, t):
    x, y, z = X[..., 0], X[..., 1], X[..., 2]
    r2 = x * x + y * y
    f = np.sin(np.pi * z) * np.cos(np.pi * t) / r2
    return np.stack([x * f, y * f, np.zeros_like(f)], -1)


def tem_B(X, t):
    x, y, z = X[..., 0], X[..., 1], X[..., 2]
    r2 = x * x + y * y
    f = np.cos(np.pi * z) * np.sin(np.pi * t) / r2
    return np.stack([y * f, -x * f, np.zeros_like(f)], -1)


def tem_spatial(X):
    """E_s with E(x, t) = cos(pi t) E_s(x): the separable Dirichlet datum."""
    return tem_E(X, 0.0)


def coax_geometry(n):
    from .workloads import quarter_annulus
    return quarter_annulus(n, r1=R1, r2=R2, height=1.0)


# ---- full-space index maps ------------------------------------------------------------------

def interior_mask(p, n, k):
    """Boolean mask over the full X^k_h (primalF) vector: True on the functions of X^k_{h,0}."""
    n = forms._n3(n)
    masks = []
    for s in forms.component_spaces("primalF", k):
        m1 = [np.ones(_dim(s[a], p, n[a]), dtype=bool) for a in range(3)]
        for a in range(3):
            if s[a] == "SpF":
                m1[a][0] = m1[a][-1] = False
        masks.append((m1[2][:, None, None] & m1[1][None, :, None] & m1[0][None, None, :]).ravel())
    return np.concatenate(masks)


def _dim(space, p, n):
    from .splines import space_dim
    return space_dim(space, p, n)


# ---- the lifting: local projection of tangential boundary data (reading Z29) ----------------

def lifting_coefficients(p, n, ctrl, E_fn, faces, Q=None):
    """e^_b in the full X^1_h: on each Dirichlet face (axis, side) in `faces`, the tangential
    covariant components e^_c(x^) = DF[:, c] . E_fn(F(x^)) projected (unweighted, parametric L2) onto
    the face trace space of component c; zero elsewhere."""
    n = forms._n3(n)
    Q = Q or p + 2
    shapes = forms.component_shapes("primalF", 1, p, n)
    comps = [np.zeros(s[::-1]) for s in shapes]     # [z][y][x]
    face_set = set(faces)
    for (ax, side) in faces:
        for c in range(3):
            if c == ax:
                continue                             # the normal component has no trace
            t = 3 - ax - c                           # the other tangential axis
            spc = forms.component_spaces("primalF", 1)[c]
            # 1D bases of the face trace space along c (own, S_{p-1}) and t (S_p full, trimmed at
            # ends whose face carries homogeneous data)
            xs, ws = gauss_rule(n[c], Q)
            ts, wt = gauss_rule(n[t], Q)
            Vc = space_values(spc[c], p, n[c], xs)
            Vt = space_values(spc[t], p, n[t], ts)
            keep = np.ones(Vt.shape[1], dtype=bool)
            if (t, 0) not in face_set:
                keep[0] = False
            if (t, 1) not in face_set:
                keep[-1] = False
            Vt = Vt[:, keep]
            # face points x^ (the face coordinate fixed), geometry there
            P = np.zeros((len(ts), len(xs), 3))
            P[..., ax] = float(side)
            P[..., c] = xs[None, :]
            P[..., t] = ts[:, None]
            F, DF = _geometry_at_points(p, n, ctrl, P.reshape(-1, 3))
            E = E_fn(F)
            g = np.einsum("qi,qi->q", DF[:, :, c], E).reshape(len(ts), len(xs))
            rhs = Vt.T @ (wt[:, None] * g * ws[None, :]) @ Vc       # [t-basis, c-basis]
            Gt = Vt.T @ (wt[:, None] * Vt)
            Gc = Vc.T @ (ws[:, None] * Vc)
            coef = np.linalg.solve(Gt, np.linalg.solve(Gc, rhs.T).T)  # Gt^{-1} rhs Gc^{-1}
            full = np.zeros((keep.size, Vc.shape[1]))
            full[keep] = coef
            # write into component c at index 0 / last along ax
            arr = comps[c]                            # [z][y][x]
            sl = [slice(None)] * 3
            sl[2 - ax] = 0 if side == 0 else -1
            face = arr[tuple(sl)]                     # remaining dims in [z][y][x] order without ax
            rem = [a for a in (2, 1, 0) if a != ax]   # array axes order (as axis ids)
            face[...] = full.T if rem == [c, t] else full
    return forms.join(comps)


def _geometry_at_points(p, n, ctrl, pts):
    """F and DF at arbitrary parametric points (rational or polynomial map)."""
    import types
    q = types.SimpleNamespace(p=p, n=n, nqp=len(pts), x1d=None)
    # evaluate point by point along a degenerate tensor grid: one point per call keeps it simple
    Fs, DFs = [], []
    for x in pts:
        q.x1d = [np.array([x[0]]), np.array([x[1]]), np.array([x[2]])]
        q.nqp = 1
        F, DF = geometry_at_qp(q, ctrl)
        Fs.append(F[0])
        DFs.append(DF[0])
    return np.array(Fs), np.array(DFs)


# ---- tier A with lifting (the paper's formulation, literally) ---------------------------------

class TierAL(TierA):
    """Scheme 2 with the lifted E: state (d, e_0, b in X^2_h, h).  Materials eps = mu = 1
    unless given at the quadrature points (element-major), as TierA."""

    def __init__(self, p, n, ctrl, e_hat_b, inv_eps_qp=None, inv_mu_qp=None, Q=None):
        super().__init__(p, n, ctrl=ctrl, inv_eps_qp=inv_eps_qp, inv_mu_qp=inv_mu_qp, Q=Q)
        self.D1F = forms.incidence("primalF", 1, p, self.n).astype(np.float64)   # X1_h -> X2_h
        self.e_int = interior_mask(p, self.n, 1)
        self.b_int = interior_mask(p, self.n, 2)
        self.K1F = _pairing_full(self.quad)                                      # X~2 x X1_h
        self.MmuF = _mass2_full_cols(self.quad, inv_mu_qp, ctrl)                 # X2_{h,0} x X2_h
        self.e_hat_b = np.asarray(e_hat_b, dtype=np.float64)
        self.N_bF = self.b_int.size

    def step(self, d, e0, bF, h, dt, g_next, jhat=None, s=1.0):
        d = d + dt * (self.Dt1 @ h - (s * jhat if jhat is not None else 0.0))
        eb = g_next * self.e_hat_b
        e0 = self.solve_K1(self.Meps @ d - self.K1F[:, ~self.e_int] @ eb[~self.e_int])   # (K1)_0 e_0 = M~2 d - (K1)_b e_b
        eF = eb.copy()
        eF[self.e_int] = e0
        bF = bF - dt * (self.D1F @ eF)                                                   # D1 : X1_h -> X2_h
        h = self.solve_Kt1(self.MmuF @ bF)                                               # M2 columns in X2_h
        return d, e0, bF, h

    def run(self, d, e0, bF, h, dt, n_steps, g_fn, t0=0.0, jhat=None, jamp=None):
        for k in range(n_steps):
            s = 1.0 if jamp is None else jamp[k]
            d, e0, bF, h = self.step(d, e0, bF, h, dt, g_fn(t0 + (k + 1) * dt), jhat, s)
        return d, e0, bF, h


def _pairing_full(quad):
    """K1 with columns in the full X^1_h: rows dual 2-forms, int eta~ ^ w."""
    R = [basis_at_qp(quad, "dual", 2, c) for c in range(3)]
    C = [basis_at_qp(quad, "primalF", 1, c) for c in range(3)]
    blocks = [[None] * 3 for _ in range(3)]
    for c in range(3):
        for c2 in range(3):
            blocks[c][c2] = (R[c].T @ sp.diags(quad.w) @ C[c]) if c == c2 else sp.csr_matrix((R[c].shape[1], C[c2].shape[1]))
    return _blocks_to_sparse(blocks)


def _mass2_full_cols(quad, gamma_qp, ctrl):
    """M2_{1/mu}: rows the primal 2-forms of X^2_{h,0}, columns the full X^2_h."""
    from .assemble import qp_elem_to_grid
    R = [basis_at_qp(quad, "primal", 2, c) for c in range(3)]
    C = [basis_at_qp(quad, "primalF", 2, c) for c in range(3)]
    _, DF = geometry_at_qp(quad, ctrl)
    det = np.linalg.det(DF)
    g = np.ones(quad.nqp) if gamma_qp is None else qp_elem_to_grid(gamma_qp, quad.n, quad.Q)
    blocks = [[None] * 3 for _ in range(3)]
    for c in range(3):
        for c2 in range(3):
            coef = np.einsum("qi,qi->q", DF[:, :, c], DF[:, :, c2]) / det * g * quad.w
            blocks[c][c2] = R[c].T @ sp.diags(coef) @ C[c2]
    return _blocks_to_sparse(blocks)


# ---- projections of 2-form data and errors on the curved map (reading Z12) ---------------------

def project_2form(p, n, ctrl, field, cplx, Q=None):
    """Unweighted parametric L2 projection of the pulled-back 2-form proxy det(DF) DF^{-1} B(F(x^))
    onto the 2-form space of complex `cplx` ('dual' = X~2, 'primalF' = X^2_h)."""
    n = forms._n3(n)
    Q = Q or p + 2
    quad = Quad(p, n, Q)
    F, DF = geometry_at_qp(quad, ctrl)
    det = np.linalg.det(DF)
    proxy = np.einsum("qij,qj->qi", np.linalg.inv(DF), field(F)) * det[:, None]
    shape = (len(quad.x1d[2]), len(quad.x1d[1]), len(quad.x1d[0]))
    out = []
    for c, spc in enumerate(forms.component_spaces(cplx, 2)):
        V = [space_values(spc[a], p, n[a], quad.x1d[a]) for a in range(3)]
        w3 = quad.w.reshape(shape)
        rhs = kron3(V[0].T, V[1].T, V[2].T, w3 * proxy[:, c].reshape(shape))
        Ginv = [np.linalg.inv(V[a].T @ (quad.w1d[a][:, None] * V[a])) for a in range(3)]
        out.append(kron3(Ginv[0], Ginv[1], Ginv[2], rhs))
    return forms.join(out)


def l2_error_1form(p, n, ctrl, cplx, v, exact, Q=None):
    """Relative L2(Omega) error of the 1-form with coefficients v (complex 'primalF' = X^1_h or
    'dual' = X~1), pushed forward E_h = DF^{-T} e^, against exact(F(x^))."""
    n = forms._n3(n)
    Q = Q or p + 2
    quad = Quad(p, n, Q)
    F, DF = geometry_at_qp(quad, ctrl)
    det = np.linalg.det(DF)
    comps = forms.split(v, cplx, 1, p, n)
    proxy = np.stack([basis_at_qp(quad, cplx, 1, c) @ comps[c].ravel() for c in range(3)], -1)
    Eh = np.einsum("qji,qj->qi", np.linalg.inv(DF), proxy)   # DF^{-T} e^
    Ex = exact(F)
    w = quad.w * det
    return np.sqrt(np.sum(w[:, None] * (Eh - Ex) ** 2) / np.sum(w[:, None] * Ex ** 2))


def coax_setup(p, n, dt, Q=None):
    """The coax TEM problem: (TierAL, initial state (d0, e0, bF^{1/2}, h^{1/2}), g(t) = cos(pi t))."""
    ctrl = coax_geometry(n)
    faces = [(1, 0), (1, 1)]
    ehb = lifting_coefficients(p, n, ctrl, tem_spatial, faces)
    A = TierAL(p, n, ctrl, ehb, Q=Q)
    g = lambda t: np.cos(np.pi * t)  # noqa: E731
    d0 = project_2form(p, n, ctrl, lambda X: tem_E(X, 0.0), "dual")
    bF = project_2form(p, n, ctrl, lambda X: tem_B(X, 0.5 * dt), "primalF")
    e0 = A.solve_K1(A.Meps @ d0 - A.K1F[:, ~A.e_int] @ (g(0.0) * ehb)[~A.e_int])
    h = A.solve_Kt1(A.MmuF @ bF)
    return A, (d0, e0, bF, h), g


def lifting_vectors(A, bF0, dt):
    """The precomputed vectors of the lifted step as sgm_step_lifted takes them (sgm.h):
    w_e = (K1)_0^{-1} (K1)_b e^_b, c_b / u_b = interior / boundary rows of D1 e^_b,
    q0 = K~1^{-1} M2_{0b} b_bnd(0), q1 = K~1^{-1} M2_{0b} u_b."""
    eb = A.e_hat_b
    w_e = A.solve_K1(A.K1F[:, ~A.e_int] @ eb[~A.e_int])
    De = A.D1F @ eb
    c_b, u_b = De[A.b_int], De[~A.b_int]
    assert np.abs((A.D1F[~A.b_int][:, A.e_int]).toarray()).max(initial=0.0) == 0.0  # D1_{b0} = 0
    Mb = A.MmuF[:, ~A.b_int]
    q0 = A.solve_Kt1(Mb @ bF0[~A.b_int])
    q1 = A.solve_Kt1(Mb @ u_b)
    return {"w_e": w_e, "c_b": c_b, "u_b": u_b, "q0": q0, "q1": q1}
