"""Tier A: scheme 2 with assembled sparse matrices and a generic sparse direct solve
(TEST INFRASTRUCTURE ONLY).

One leapfrog step, exactly eqs. discrete2_ampere / hodge_eps / faraday / hodge_mu
(P:L369-372), with d, e at t_n and b, h at t_{n+1/2} (reading Z8):

    d <- d + dt (D~1 h - s j)           (source j in X~2 with dJ = 0)
    e <- K1^{-1} (M~2_{1/eps} d)
    b <- b - dt D1 e
    h <- K~1^{-1} (M2_{1/mu} b)

K1 and K~1 are block diagonal; each diagonal block is factored once by SuperLU
(scipy.sparse.linalg.splu, with its own pivoting) and reused.
"""
import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from . import forms
from .assemble import Quad, pairing, mass1, mass2


class TierA:
    def __init__(self, p, n, ctrl=None, inv_eps_qp=None, inv_mu_qp=None, Q=None):
        self.p = p
        self.n = forms._n3(n)
        self.quad = Quad(p, self.n, Q)
        self.ctrl = ctrl
        self.D1 = forms.incidence("primal", 1, p, self.n)      # X1_{h,0} -> X2_{h,0}
        self.Dt1 = forms.incidence("dual", 1, p, self.n)       # X~1 -> X~2
        self.D2 = forms.incidence("primal", 2, p, self.n)
        self.Dt2 = forms.incidence("dual", 2, p, self.n)
        self.K1 = pairing(self.quad, "K1")
        self.Kt1 = pairing(self.quad, "Kt1")
        self.Meps = mass2(self.quad, "dual", inv_eps_qp, ctrl)     # M~2_{1/eps}
        self.Mmu = mass2(self.quad, "primal", inv_mu_qp, ctrl)     # M2_{1/mu}
        self.off_e = forms.offsets("primal", 1, p, self.n)
        self.off_h = forms.offsets("dual", 1, p, self.n)
        self._lu_K1 = [spla.splu(self.K1[self.off_e[c]:self.off_e[c + 1],
                                         self.off_e[c]:self.off_e[c + 1]].tocsc()) for c in range(3)]
        self._lu_Kt1 = [spla.splu(self.Kt1[self.off_h[c]:self.off_h[c + 1],
                                           self.off_h[c]:self.off_h[c + 1]].tocsc()) for c in range(3)]
        self.N_e = self.off_e[-1]
        self.N_h = self.off_h[-1]

    # --- Kronecker-block solves by generic sparse direct LU ----------------------------------
    def solve_K1(self, r, transpose=False):
        o = self.off_e
        return np.concatenate([self._lu_K1[c].solve(r[o[c]:o[c + 1]], trans="T" if transpose else "N")
                               for c in range(3)])

    def solve_Kt1(self, r, transpose=False):
        o = self.off_h
        return np.concatenate([self._lu_Kt1[c].solve(r[o[c]:o[c + 1]], trans="T" if transpose else "N")
                               for c in range(3)])

    # --- the step ----------------------------------------------------------------------------
    def step(self, d, e, b, h, dt, jhat=None, s=1.0):
        d = d + dt * (self.Dt1 @ h - (s * jhat if jhat is not None else 0.0))
        e = self.solve_K1(self.Meps @ d)
        b = b - dt * (self.D1 @ e)
        h = self.solve_Kt1(self.Mmu @ b)
        return d, e, b, h

    def run(self, d, e, b, h, dt, n_steps, jhat=None, jamp=None):
        for k in range(n_steps):
            s = 1.0 if jamp is None else jamp[k]
            d, e, b, h = self.step(d, e, b, h, dt, jhat, s)
        return d, e, b, h

    # --- diagnostics -------------------------------------------------------------------------
    def energy(self, d, e, b, h):
        """E_h = 1/2 (d^T K1 e + b^T K~1 h)  -- eq. energy_matrix_wedge rewritten with
        K~2 = K1^T and K2 = K~1^T."""
        return 0.5 * (d @ (self.K1 @ e) + b @ (self.Kt1 @ h))

    def gauss(self, d, b):
        """(||D~2 d||_inf, ||D2 b||_inf): discrete Gauss laws."""
        return float(np.max(np.abs(self.Dt2 @ d), initial=0.0)), float(np.max(np.abs(self.D2 @ b), initial=0.0))


class TierA1(TierA):
    """Tier A of the FIRST scheme (eqs. discrete1_*): the Hodge stars solve the 1-form
    mass matrices,
        M^1_eps e = K~2 d,     M~^1_mu h = K2 b,      K~2 = K1^T, K2 = K~1^T,
    by SuperLU on the assembled masses; Ampere / Faraday updates as in scheme 2.  eps_qp, mu_qp:
    the materials themselves (not their inverses) at the quadrature points, element-major."""

    def __init__(self, p, n, ctrl=None, eps_qp=None, mu_qp=None, Q=None):
        super().__init__(p, n, ctrl=ctrl, Q=Q)
        self.M1eps = mass1(self.quad, "primal", eps_qp, ctrl)
        self.M1mu = mass1(self.quad, "dual", mu_qp, ctrl)
        self._lu_M1eps = spla.splu(self.M1eps.tocsc())
        self._lu_M1mu = spla.splu(self.M1mu.tocsc())

    def hodge_eps(self, d):
        return self._lu_M1eps.solve(self.K1.T @ d)        # eq. discrete1_hodge_eps

    def hodge_mu(self, b):
        return self._lu_M1mu.solve(self.Kt1.T @ b)        # eq. discrete1_hodge_mu

    def step(self, d, e, b, h, dt, jhat=None, s=1.0):
        d = d + dt * (self.Dt1 @ h - (s * jhat if jhat is not None else 0.0))   # eq. discrete1_ampere
        e = self.hodge_eps(d)
        b = b - dt * (self.D1 @ e)                                            # eq. discrete1_faraday
        h = self.hodge_mu(b)
        return d, e, b, h
