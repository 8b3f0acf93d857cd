"""Tier B: the scheme-2 step through the paper's own Kronecker identities
(TEST INFRASTRUCTURE ONLY; pinned against tier A in tests/test_oracle_tierb.py).

* 1D factors: Hat{G} = int D''_k B_c (dual S_{p-2} CS rows, primal S_p cols) and
  Hat{M} = int B'_j D'_k (dual S_{p-1} B-spline rows, primal S_{p-1} CS cols), from
  ``splines.gram_1d``.
* K1 blocks C_c (eq. tensor_K): Hat{M} along axis c, Hat{G} along the others.
  K~1 blocks (eq. tensor_Ktilde): Hat{G}^T along axis c, Hat{M}^T along the others.
* Inverse (eq. kroninverse) applied mode by mode with the vec trick:
  one dense 1D inverse per axis, applied with np.tensordot along that axis.
* Masses: separable case (identity / axis-aligned affine F, constant material) as Kronecker
  products of 1D Grams; general case by sum factorisation on the global quadrature grid
  (interpolate -> multiply by W -> test), the same (p+1)-point rule as tier A (reading Z13).
* Curls via slicing differences (the Cartesian incidence structure).
"""
import numpy as np

from . import forms
from .splines import gram_1d, space_values, open_knots, bspline_values, bspline_derivatives
from .assemble import Quad, qp_elem_to_grid, Rational


def apply_axis(A, X, axis):
    """Apply matrix A along `axis` of the [z][y][x] array X (axis 0=x, 1=y, 2=z)."""
    ax = 2 - axis
    return np.moveaxis(np.tensordot(A, X, axes=([1], [ax])), 0, ax)


def kron3(Ax, Ay, Az, X):
    """(Az (x) Ay (x) Ax) vec(X) for X shaped [z][y][x]."""
    return apply_axis(Az, apply_axis(Ay, apply_axis(Ax, X, 0), 1), 2)


# --- 1D curls on component arrays -----------------------------------------------------------

def _dprimal(u, axis):
    """(du)_j = u_j - u_{j-1} with u_{-1} = u_a = 0 along axis (primal, trimmed)."""
    ax = 2 - axis
    pad = [(0, 0)] * 3
    pad[ax] = (1, 1)
    up = np.pad(u, pad)
    return np.diff(up, axis=ax)


def _ddual(v, axis):
    """(dv)_j = v_{j+1} - v_j along axis (dual, free)."""
    return np.diff(v, axis=2 - axis)


def curl_primal(e):
    e1, e2, e3 = e
    return [_dprimal(e3, 1) - _dprimal(e2, 2), _dprimal(e1, 2) - _dprimal(e3, 0), _dprimal(e2, 0) - _dprimal(e1, 1)]


def curl_dual(h):
    h1, h2, h3 = h
    return [_ddual(h3, 1) - _ddual(h2, 2), _ddual(h1, 2) - _ddual(h3, 0), _ddual(h2, 0) - _ddual(h1, 1)]


def div_primal(b):
    return _dprimal(b[0], 0) + _dprimal(b[1], 1) + _dprimal(b[2], 2)


def div_dual(d):
    return _ddual(d[0], 0) + _ddual(d[1], 1) + _ddual(d[2], 2)


class TierB:
    """Structured oracle.  Materials: ``inv_eps`` / ``inv_mu`` are either a float (constant)
    or per-quadrature-point arrays (element-major layout); ``ctrl`` None = identity map."""

    def __init__(self, p, n, ctrl=None, inv_eps=1.0, inv_mu=1.0, Q=None):
        self.p = p
        self.n = forms._n3(n)
        self.Q = Q if Q is not None else p + 1
        self.ctrl = ctrl
        n3 = self.n
        self.G = [gram_1d("Dp2", "Sp", p, n3[a]) for a in range(3)]
        self.M = [gram_1d("Dp1", "Sp1", p, n3[a]) for a in range(3)]
        self.Ginv = [np.linalg.inv(G) for G in self.G]
        self.Minv = [np.linalg.inv(M) for M in self.M]
        self.GamB1 = [gram_1d("Dp1", "Dp1", p, n3[a]) for a in range(3)]   # Gamma_B^{p-1}
        self.GamC2 = [gram_1d("Dp2", "Dp2", p, n3[a]) for a in range(3)]   # Gamma_C^{p-2}
        self.GamBp = [gram_1d("Sp", "Sp", p, n3[a]) for a in range(3)]     # Gamma_B^{p}
        self.GamC1 = [gram_1d("Sp1", "Sp1", p, n3[a]) for a in range(3)]   # Gamma_C^{p-1}
        self.sh_e = forms.component_shapes("primal", 1, p, n3)
        self.sh_h = forms.component_shapes("dual", 1, p, n3)
        self.N_e = forms.form_dim("primal", 1, p, n3)
        self.N_h = forms.form_dim("dual", 1, p, n3)
        self.sep_eps = self._separable(inv_eps)
        self.sep_mu = self._separable(inv_mu)
        self.inv_eps = inv_eps
        self.inv_mu = inv_mu
        if self.sep_eps is None:
            self.W_eps = self._W(inv_eps)
        if self.sep_mu is None:
            self.W_mu = self._W(inv_mu)

    # --- geometry / W ---------------------------------------------------------------------
    def _separable(self, gamma):
        """Per-component constant scale if the Hodge is separable, else None."""
        if not np.isscalar(gamma):
            return None
        if self.ctrl is None:
            return np.array([gamma] * 3, dtype=np.float64)
        return None

    def _geometry(self):
        """DF on the global quadrature grid by sum factorisation; a ``Rational`` map uses the
        quotient rule on numerator sum w P B and denominator sum w B."""
        quad = Quad(self.p, self.n, self.Q)
        shp = (self.n[2] + self.p, self.n[1] + self.p, self.n[0] + self.p)
        V, D = [], []
        for a in range(3):
            X = open_knots(self.p, self.n[a])
            V.append(bspline_values(X, self.p, quad.x1d[a]))
            D.append(bspline_derivatives(X, self.p, quad.x1d[a]))
        DF = np.empty((len(quad.x1d[2]), len(quad.x1d[1]), len(quad.x1d[0]), 3, 3))
        if isinstance(self.ctrl, Rational):
            w = self.ctrl.w.reshape(shp)
            wP = self.ctrl.P.reshape(shp + (3,)) * w[..., None]
            Wq = kron3(V[0], V[1], V[2], w)
            dW = [kron3(D[0], V[1], V[2], w), kron3(V[0], D[1], V[2], w), kron3(V[0], V[1], D[2], w)]
            for i in range(3):
                C = wP[..., i]
                Fi = kron3(V[0], V[1], V[2], C) / Wq
                DF[..., i, 0] = (kron3(D[0], V[1], V[2], C) - Fi * dW[0]) / Wq
                DF[..., i, 1] = (kron3(V[0], D[1], V[2], C) - Fi * dW[1]) / Wq
                DF[..., i, 2] = (kron3(V[0], V[1], D[2], C) - Fi * dW[2]) / Wq
            return quad, DF
        ctrl = np.asarray(self.ctrl, dtype=np.float64).reshape(shp + (3,))
        for i in range(3):
            C = ctrl[..., i]
            DF[..., i, 0] = kron3(D[0], V[1], V[2], C)
            DF[..., i, 1] = kron3(V[0], D[1], V[2], C)
            DF[..., i, 2] = kron3(V[0], V[1], D[2], C)
        return quad, DF

    def _W(self, gamma):
        """W_{cc'}(q) = w_q gamma(q) (DF^T DF)_{cc'} / det DF on the global quadrature grid."""
        quad = Quad(self.p, self.n, self.Q)
        shape = (len(quad.x1d[2]), len(quad.x1d[1]), len(quad.x1d[0]))
        g = np.broadcast_to(np.asarray(gamma, dtype=np.float64), ()) if np.isscalar(gamma) else None
        gq = (np.full(shape, float(gamma)) if g is not None
              else qp_elem_to_grid(gamma, self.n, self.Q).reshape(shape))
        w = quad.w.reshape(shape)
        if self.ctrl is None:
            return {"diag": w * gq}
        _, DF = self._geometry()
        det = np.linalg.det(DF)
        G = np.einsum("...ki,...kj->...ij", DF, DF) / det[..., None, None]
        return {"full": G * (w * gq)[..., None, None]}

    # --- masses ---------------------------------------------------------------------------
    def _mass(self, comps, cplx, sep, W, own, other):
        p, n = self.p, self.n
        if sep is not None:
            out = []
            for c in range(3):
                A = [own[a] if a == c else other[a] for a in range(3)]
                out.append(sep[c] * kron3(A[0], A[1], A[2], comps[c]))
            return out
        quad = Quad(p, n, self.Q)
        sp2 = forms.component_spaces(cplx, 2)
        V = [[space_values(sp2[c][a], p, n[a], quad.x1d[a]) for a in range(3)] for c in range(3)]
        u = [kron3(V[c][0], V[c][1], V[c][2], comps[c]) for c in range(3)]
        if "diag" in W:
            v = [W["diag"] * u[c] for c in range(3)]
        else:
            F = W["full"]
            v = [sum(F[..., c, c2] * u[c2] for c2 in range(3)) for c in range(3)]
        return [kron3(V[c][0].T, V[c][1].T, V[c][2].T, v[c]) for c in range(3)]

    def mass_eps(self, d):
        """M~2_{1/eps} d."""
        sep = self.sep_eps
        return self._mass(d, "dual", sep, None if sep is not None else self.W_eps, self.GamB1, self.GamC2)

    def mass_mu(self, b):
        """M2_{1/mu} b."""
        sep = self.sep_mu
        return self._mass(b, "primal", sep, None if sep is not None else self.W_mu, self.GamBp, self.GamC1)

    # --- pairings ------------------------------------------------------------------------------
    def _K1_factors(self, c, inv=False, T=False):
        own = (self.Minv if inv else self.M)
        oth = (self.Ginv if inv else self.G)
        A = [own[a] if a == c else oth[a] for a in range(3)]
        return [x.T for x in A] if T else A

    def _Kt1_factors(self, c, inv=False, T=False):
        # K~1 block c: Hat{G}^T along own axis, Hat{M}^T along others
        own = [(Gi.T) for Gi in (self.Ginv if inv else self.G)]
        oth = [(Mi.T) for Mi in (self.Minv if inv else self.M)]
        A = [own[a] if a == c else oth[a] for a in range(3)]
        return [x.T for x in A] if T else A

    def apply_K1(self, e, T=False):
        return [kron3(*self._K1_factors(c, T=T), e[c]) for c in range(3)]

    def apply_Kt1(self, h, T=False):
        return [kron3(*self._Kt1_factors(c, T=T), h[c]) for c in range(3)]

    def solve_K1(self, r, T=False):
        return [kron3(*self._K1_factors(c, inv=True, T=T), r[c]) for c in range(3)]

    def solve_Kt1(self, r, T=False):
        return [kron3(*self._Kt1_factors(c, inv=True, T=T), r[c]) for c in range(3)]

    # --- step ----------------------------------------------------------------------------------
    def split_e(self, v):
        return forms.split(v, "primal", 1, self.p, self.n)

    def split_h(self, v):
        return forms.split(v, "dual", 1, self.p, self.n)

    def step(self, d, e, b, h, dt, jhat=None, s=1.0):
        """One leapfrog step on flat vectors; returns flat vectors."""
        d, b, h = self.split_e(d), self.split_h(b), self.split_h(h)
        cd = curl_dual(h)
        if jhat is not None:
            j = self.split_e(jhat)
            d = [d[c] + dt * (cd[c] - s * j[c]) for c in range(3)]
        else:
            d = [d[c] + dt * cd[c] for c in range(3)]
        e = self.solve_K1(self.mass_eps(d))
        ce = curl_primal(e)
        b = [b[c] - dt * ce[c] for c in range(3)]
        h = self.solve_Kt1(self.mass_mu(b))
        return forms.join(d), forms.join(e), forms.join(b), forms.join(h)

    def run(self, d, e, b, h, dt, n_steps, jhat=None, jamp=None):
        for k in range(n_steps):
            s = 1.0 if jamp is None else jamp[k]
            d, e, b, h = self.step(d, e, b, h, dt, jhat, s)
        return d, e, b, h

    def step_eh(self, e, h, dt, jhat=None, s=1.0):
        """The (e,h)-state form of one step (the Petrov-Galerkin scheme in E_h, H_h, P:L395-408,
        with its typos corrected per reading Z6): e <- e + K1^{-1} M~2_{1/eps} (dt (D~1 h - s j)),
        h <- h - K~1^{-1} M2_{1/mu} (dt D1 e); the same as step() on e = K1^{-1} M~2 d,
        h = K~1^{-1} M2 b (eqs. discrete2_*), d and b never formed."""
        cd = curl_dual(self.split_h(h))
        if jhat is not None:
            j = self.split_e(jhat)
            r = [dt * (cd[c] - s * j[c]) for c in range(3)]
        else:
            r = [dt * cd[c] for c in range(3)]
        e = e + forms.join(self.solve_K1(self.mass_eps(r)))
        ce = curl_primal(self.split_e(e))
        h = h - forms.join(self.solve_Kt1(self.mass_mu([dt * ce[c] for c in range(3)])))
        return e, h

    def run_eh(self, e, h, dt, n_steps, jhat=None, jamp=None):
        for k in range(n_steps):
            e, h = self.step_eh(e, h, dt, jhat, 1.0 if jamp is None else jamp[k])
        return e, h

    def hodge_eps(self, d):
        """e = K1^{-1} M~2_{1/eps} d  (eq. discrete2_hodge_eps)."""
        return forms.join(self.solve_K1(self.mass_eps(self.split_e(d))))

    def hodge_mu(self, b):
        """h = K~1^{-1} M2_{1/mu} b  (eq. discrete2_hodge_mu)."""
        return forms.join(self.solve_Kt1(self.mass_mu(self.split_h(b))))

    def energy(self, d, e, b, h):
        """1/2 (d^T K1 e + b^T K~1 h)."""
        K1e = forms.join(self.apply_K1(self.split_e(e)))
        Kt1h = forms.join(self.apply_Kt1(self.split_h(h)))
        return 0.5 * (d @ K1e + b @ Kt1h)

    def gauss(self, d, b):
        return (float(np.max(np.abs(div_dual(self.split_e(d))), initial=0.0)),
                float(np.max(np.abs(div_primal(self.split_h(b))), initial=0.0)))


class TierB1(TierB):
    """Tier B of the first scheme for separable Hodge stars (identity map, constant eps, mu):
    M^1_eps and M~^1_mu are Kronecker products of 1D Grams (primal 1-forms: Gamma of the CS basis of
    S_{p-1} along the own axis, Gamma of trimmed S_p along the others; dual 1-forms: Gamma of the CS
    basis of S_{p-2} own, Gamma of S_{p-1} B-splines others), inverted mode by mode with dense 1D
    inverses; e = M^1_eps^{-1} K1^T d, h = M~^1_mu^{-1} K~1^T b."""

    def __init__(self, p, n, eps=1.0, mu=1.0, Q=None):
        super().__init__(p, n, Q=Q)
        self.eps, self.mu = float(eps), float(mu)
        self.GCinv1 = [np.linalg.inv(G) for G in self.GamC1]
        self.GBinvp = [np.linalg.inv(G) for G in self.GamBp]
        self.GCinv2 = [np.linalg.inv(G) for G in self.GamC2]
        self.GBinv1 = [np.linalg.inv(G) for G in self.GamB1]

    def hodge_eps(self, d):
        r = self.apply_K1(self.split_e(d), T=True)
        out = []
        for c in range(3):
            A = [self.GCinv1[a] if a == c else self.GBinvp[a] for a in range(3)]
            out.append(kron3(A[0], A[1], A[2], r[c]) / self.eps)
        return forms.join(out)

    def hodge_mu(self, b):
        r = self.apply_Kt1(self.split_h(b), T=True)
        out = []
        for c in range(3):
            A = [self.GCinv2[a] if a == c else self.GBinv1[a] for a in range(3)]
            out.append(kron3(A[0], A[1], A[2], r[c]) / self.mu)
        return forms.join(out)

    def step(self, d, e, b, h, dt, jhat=None, s=1.0):
        dd, bb = self.split_e(d), self.split_h(b)
        cd = curl_dual(self.split_h(h))
        if jhat is not None:
            j = self.split_e(jhat)
            dd = [dd[c] + dt * (cd[c] - s * j[c]) for c in range(3)]
        else:
            dd = [dd[c] + dt * cd[c] for c in range(3)]
        d = forms.join(dd)
        e = self.hodge_eps(d)
        ce = curl_primal(self.split_e(e))
        b = forms.join([bb[c] - dt * ce[c] for c in range(3)])
        h = self.hodge_mu(b)
        return d, e, b, h
