"""Closed-form cavity modes, projections, CFL, and the BASELINE.json configs C1-C5
(TEST INFRASTRUCTURE ONLY).

All of this is oracle-side setup: it produces the seeded inputs that both the oracle and the
GPU path consume (d, e, b, h, j^, materials at quadrature points, geometry control points, dt).
Random draws come from ``synth`` (no method arithmetic there).
"""
import numpy as np
from scipy.sparse.linalg import LinearOperator, eigs

import synth
from . import forms
from .splines import gauss_rule, space_values, open_knots, bspline_values
from .structured import TierB, kron3, apply_axis, curl_dual
from .assemble import Rational

# ------------------------------------------------------------------------------------------
# cavity eigenmodes of the unit cube with PEC walls (readings Z10, Z11)
# ------------------------------------------------------------------------------------------


class CavityMode:
    """E = alpha * (A1 c s s, A2 s c s, A3 s s c) cos(w t), k = pi m, w = pi |m|, A . m = 0;
    B = H = -(alpha/w) (k x A) (s c c, c s c, c c s) sin(w t)   (eps = mu = 1).
    Here "c s s" = cos(k1 x) sin(k2 y) sin(k3 z) etc.  The first cube mode is
    m = (1,1,0), A = (0,0,1): E = (0,0,sin pi x sin pi y) cos(sqrt2 pi t) (reading Z11)."""

    def __init__(self, m, A, alpha=1.0):
        self.m = np.asarray(m, dtype=np.float64)
        self.A = np.asarray(A, dtype=np.float64)
        if abs(self.A @ self.m) > 1e-14:
            raise ValueError("A must be orthogonal to m (divergence-free)")
        self.k = np.pi * self.m
        self.w = np.pi * np.linalg.norm(self.m)
        self.alpha = alpha

    def _trig(self, X):
        x, y, z = X[..., 0], X[..., 1], X[..., 2]
        k1, k2, k3 = self.k
        s = [np.sin(k1 * x), np.sin(k2 * y), np.sin(k3 * z)]
        c = [np.cos(k1 * x), np.cos(k2 * y), np.cos(k3 * z)]
        return s, c

    def E(self, X, t):
        s, c = self._trig(X)
        f = [c[0] * s[1] * s[2], s[0] * c[1] * s[2], s[0] * s[1] * c[2]]
        return self.alpha * np.cos(self.w * t) * np.stack([self.A[i] * f[i] for i in range(3)], -1)

    def B(self, X, t):
        s, c = self._trig(X)
        g = [s[0] * c[1] * c[2], c[0] * s[1] * c[2], c[0] * c[1] * s[2]]
        kxA = np.cross(self.k, self.A)
        return -(self.alpha / self.w) * np.sin(self.w * t) * np.stack([kxA[i] * g[i] for i in range(3)], -1)


class ModeSum:
    def __init__(self, modes):
        self.modes = modes

    def E(self, X, t):
        return sum(m.E(X, t) for m in self.modes)

    def B(self, X, t):
        return sum(m.B(X, t) for m in self.modes)


def c2_modes():
    """The four modes of configs[1] with alpha = rng(2).uniform(-1,1,4)."""
    al = synth.c2_amplitudes()
    spec = [((1, 1, 0), (0, 0, 1)), ((1, 0, 1), (0, 1, 0)), ((0, 1, 1), (1, 0, 0)),
            ((1, 1, 1), np.array([1, 1, -2]) / np.sqrt(6))]
    return ModeSum([CavityMode(m, A, a) for (m, A), a in zip(spec, al)])


# ------------------------------------------------------------------------------------------
# quadrature grid helpers (identity geometry unless noted)
# ------------------------------------------------------------------------------------------

def qp_grid(p, n, Q=None):
    """1D Gauss points/weights per axis and the 3D grid of points [z][y][x][3]."""
    n = forms._n3(n)
    Q = Q or p + 1
    xs, ws = zip(*[gauss_rule(n[a], Q) for a in range(3)])
    Z, Y, X = np.meshgrid(xs[2], xs[1], xs[0], indexing="ij")
    return xs, ws, np.stack([X, Y, Z], -1)


def grid_to_elem(arr3, n, Q):
    """[NQz][NQy][NQx] grid array -> element-major flat layout [ez][ey][ex][qz][qy][qx]."""
    nx, ny, nz = forms._n3(n)
    return np.asarray(arr3).reshape(nz, Q, ny, Q, nx, Q).transpose(0, 2, 4, 1, 3, 5).reshape(-1)


def physical_points(p, n, ctrl=None, Q=None):
    """F(x_q) on the global grid [z][y][x][3], by sum factorisation of the spline map."""
    n = forms._n3(n)
    Q = Q or p + 1
    xs, _, Xg = qp_grid(p, n, Q)
    if ctrl is None:
        return Xg
    V = [bspline_values(open_knots(p, n[a]), p, xs[a]) for a in range(3)]
    shp = (n[2] + p, n[1] + p, n[0] + p)
    if isinstance(ctrl, Rational):
        w = ctrl.w.reshape(shp)
        Wq = kron3(V[0], V[1], V[2], w)
        wP = ctrl.P.reshape(shp + (3,)) * w[..., None]
        return np.stack([kron3(V[0], V[1], V[2], wP[..., i]) / Wq for i in range(3)], -1)
    ctrl = np.asarray(ctrl, dtype=np.float64).reshape(shp + (3,))
    return np.stack([kron3(V[0], V[1], V[2], ctrl[..., i]) for i in range(3)], -1)


# ------------------------------------------------------------------------------------------
# quarter-annulus (coaxial-cable cross-section) geometry: a degree-2 NURBS map (NEXT #2 input)
# ------------------------------------------------------------------------------------------

def insert_knot(U, p, Pw, u):
    """Boehm's knot insertion on a curve with homogeneous control points Pw [m][d] (weights last):
    the curve is unchanged, one more control point (The NURBS Book, algorithm A5.1)."""
    U = np.asarray(U, dtype=np.float64)
    k = np.searchsorted(U, u, side="right") - 1
    m = len(Pw)
    Q = np.zeros((m + 1, Pw.shape[1]))
    for i in range(m + 1):
        if i <= k - p:
            Q[i] = Pw[i]
        elif i >= k + 1:
            Q[i] = Pw[i - 1]
        else:
            a = (u - U[i]) / (U[i + p] - U[i])
            Q[i] = a * Pw[i] + (1 - a) * Pw[i - 1]
    return np.insert(U, k + 1, u), Q


def quarter_annulus(n, r1=0.5, r2=1.0, height=1.0):
    """Rational degree-2 map of (0,1)^3 onto {r1 <= r <= r2, 0 <= theta <= pi/2, 0 <= z <= height}:
    x^ -> radius r1 + (r2 - r1) x^ (affine), y^ -> angle along the exact NURBS quarter circle
    (control points (1,0), (1,1), (0,1), weights 1, 1/sqrt2, 1), z^ -> z (affine); the circle is
    refined to n_y elements by knot insertion, the affine directions use Greville points.  The
    order (radial, angular, axial) gives det DF > 0.  Returns a ``Rational`` for p = 2."""
    n = forms._n3(n)
    p = 2
    U = np.array([0.0, 0, 0, 1, 1, 1])
    Pw = np.array([[1.0, 0.0, 1.0], [1.0, 1.0, 1.0], [0.0, 1.0, 1.0]])
    Pw[:, :2] *= Pw[:, 2:3] * np.array([[1.0], [1.0 / np.sqrt(2.0)], [1.0]])
    Pw[1, 2] = 1.0 / np.sqrt(2.0)
    for k in range(1, n[1]):
        U, Pw = insert_knot(U, p, Pw, k / n[1])
    arc_w = Pw[:, 2]
    arc = Pw[:, :2] / arc_w[:, None]
    g = [np.array([open_knots(p, n[a])[i + 1:i + p + 1].mean() for i in range(n[a] + p)]) for a in (0, 2)]
    r = r1 + (r2 - r1) * g[0]
    z = height * g[1]
    P = np.zeros((n[2] + p, n[1] + p, n[0] + p, 3))
    P[..., 0] = r[None, None, :] * arc[None, :, 0:1]
    P[..., 1] = r[None, None, :] * arc[None, :, 1:2]
    P[..., 2] = z[:, None, None]
    w = np.broadcast_to(arc_w[None, :, None], (n[2] + p, n[1] + p, n[0] + p)).copy()
    return Rational(P, w)


def interpolate_map(p, n, fmap):
    """Control points of the spline map in S_p(Xi)^3 interpolating fmap at the Greville
    points (reading Z18).  fmap: X[...,3] -> F[...,3]."""
    n = forms._n3(n)
    gs, Bs = [], []
    for a in range(3):
        X = open_knots(p, n[a])
        g = np.array([X[i + 1:i + p + 1].mean() for i in range(n[a] + p)])
        gs.append(g)
        Bs.append(bspline_values(X, p, g))
    Z, Y, Xg = np.meshgrid(gs[2], gs[1], gs[0], indexing="ij")
    F = fmap(np.stack([Xg, Y, Z], -1))
    inv = [np.linalg.inv(B) for B in Bs]
    return np.stack([kron3(inv[0], inv[1], inv[2], F[..., i]) for i in range(3)], -1)


def c3_map(X):
    """C3 map: x -> x + 0.1 sin(pi x) sin(pi y) sin(pi z) (1,1,1) (BASELINE.json configs[2])."""
    s = 0.1 * np.sin(np.pi * X[..., 0]) * np.sin(np.pi * X[..., 1]) * np.sin(np.pi * X[..., 2])
    return X + s[..., None]


# ------------------------------------------------------------------------------------------
# L2 projections (unweighted, parametric = physical for the identity map; reading Z12)
# ------------------------------------------------------------------------------------------

def _project(p, n, cplx, k, field_grid, Q=None):
    """Unweighted L2 projection of a k-form given by its proxy components on the global
    quadrature grid ([z][y][x][3]) onto the component spaces: Gram solve per component."""
    n = forms._n3(n)
    Q = Q or p + 1
    xs, ws, _ = qp_grid(p, n, Q)
    spaces = forms.component_spaces(cplx, k)
    out = []
    for c, sc in enumerate(spaces):
        V = [space_values(sc[a], p, n[a], xs[a]) for a in range(3)]
        w3 = ws[2][:, None, None] * ws[1][None, :, None] * ws[0][None, None, :]
        rhs = kron3(V[0].T, V[1].T, V[2].T, w3 * field_grid[..., c])
        Ginv = [np.linalg.inv(V[a].T @ (ws[a][:, None] * V[a])) for a in range(3)]
        out.append(kron3(Ginv[0], Ginv[1], Ginv[2], rhs))
    return forms.join(out)


def project_dual2(p, n, field_grid, Q=None):
    return _project(p, n, "dual", 2, field_grid, Q)


def project_primal2(p, n, field_grid, Q=None):
    return _project(p, n, "primal", 2, field_grid, Q)


def project_dual1(p, n, field_grid, Q=None):
    return _project(p, n, "dual", 1, field_grid, Q)


def eval_form(p, n, cplx, k, v, Q=None):
    """Parametric proxy of the discrete form v at the global quadrature grid [z][y][x][3]."""
    n = forms._n3(n)
    Q = Q or p + 1
    xs, _, _ = qp_grid(p, n, Q)
    comps = forms.split(v, cplx, k, p, n)
    out = []
    for c, sc in enumerate(forms.component_spaces(cplx, k)):
        V = [space_values(sc[a], p, n[a], xs[a]) for a in range(3)]
        out.append(kron3(V[0], V[1], V[2], comps[c]))
    return np.stack(out, -1)


def l2_rel_error(p, n, cplx, k, v, exact_grid, Q=None):
    n = forms._n3(n)
    Q = Q or p + 1
    _, ws, _ = qp_grid(p, n, Q)
    w3 = ws[2][:, None, None] * ws[1][None, :, None] * ws[0][None, None, :]
    diff = eval_form(p, n, cplx, k, v, Q) - exact_grid
    return np.sqrt(np.sum(w3[..., None] * diff ** 2) / np.sum(w3[..., None] * exact_grid ** 2))


# ------------------------------------------------------------------------------------------
# CFL (reading Z15: dt_max = 2 / sqrt(lambda_max(D~1 K~1^{-1} M2 D1 K1^{-1} M~2)))
# ------------------------------------------------------------------------------------------

def cfl_dt_max(tb: TierB, tol=1e-8):
    """Leapfrog stability limit of scheme 2 (parity unpinned in absolute value, Z15).

    d^{n+1} - 2 d^n + d^{n-1} = -dt^2 A d^n with A = D~1 K~1^{-1} M2 D1 K1^{-1} M~2, stable iff
    dt^2 lambda_max(A) < 4.  lambda_max by ARPACK (a library eigen-solver) on A.
    """
    from .structured import curl_primal

    def A(x):
        d = tb.split_e(np.asarray(x).ravel())
        e = tb.solve_K1(tb.mass_eps(d))
        b = curl_primal(e)
        h = tb.solve_Kt1(tb.mass_mu(b))
        return forms.join(curl_dual(h))

    N = tb.N_e
    op = LinearOperator((N, N), matvec=A, dtype=np.float64)
    v0 = synth.rng(100).standard_normal(N)
    lam = eigs(op, k=1, which="LM", v0=v0, tol=tol, return_eigenvectors=False)
    lam = float(np.max(np.real(lam)))
    return 2.0 / np.sqrt(lam)


def cfl_power(tb, x0, n_iter):
    """Power iteration for the same lambda_max, in the form SURVEY 8(d) fixes for reproducible dt
    ("start vector rng(100+k), 300 iterations, Rayleigh quotient"; K8, NEXT #3).

    A = D~1 K~1^{-1} M2 D1 K1^{-1} M~2 is self-adjoint and positive semi-definite in the M~2 inner
    product: K1^T D~1 = D1^T K~1 (the pairing identity behind eq. P:L240) gives
    M~2 A = C^T M2 C with C = D1 K1^{-1} M~2.  The Rayleigh quotient in that inner product is
    x.M~2 A x / x.M~2 x = (b.K~1 h) / (x.K1 e) with e = K1^{-1} M~2 x, b = D1 e,
    h = K~1^{-1} M2 b (K1 e = M~2 x, K~1 h = M2 b).  Each iteration:
        e = K1^{-1} M~2 x;  b = D1 e;  h = K~1^{-1} M2 b;
        lam_k = (b.K~1 h) / (x.K1 e);   y = D~1 h;   x = y / |y|_2
    after normalising x0 to unit 2-norm.  Works with tier A or tier B (`tb` needs solve_K1,
    solve_Kt1, mass_eps/mass_mu or Meps/Mmu, K1/Kt1 applies and the curls).
    Returns (lam_{n_iter-1}, 2/sqrt(lam), x_{n_iter}, [lam_0 .. lam_{n_iter-1}])."""
    hodge_eps, hodge_mu, K1e, Kt1h, D1, Dt1 = _ops(tb)
    x = np.asarray(x0, dtype=np.float64) / np.sqrt(np.dot(x0, x0))
    lams = []
    for _ in range(n_iter):
        e = hodge_eps(x)
        b = D1(e)
        h = hodge_mu(b)
        lams.append(float(np.dot(b, Kt1h(h)) / np.dot(x, K1e(e))))
        y = Dt1(h)
        x = y / np.sqrt(np.dot(y, y))
    lam = lams[-1]
    return lam, 2.0 / np.sqrt(lam), x, lams


def _ops(tb):
    """(e <- K1^{-1}M~2 x, h <- K~1^{-1}M2 b, K1 e, K~1 h, D1, D~1) for tier A or tier B."""
    if hasattr(tb, "Meps"):  # tier A: assembled sparse matrices (TierA1: the scheme-1 stars)
        he = tb.hodge_eps if hasattr(tb, "hodge_eps") else (lambda x: tb.solve_K1(tb.Meps @ x))
        hm = tb.hodge_mu if hasattr(tb, "hodge_mu") else (lambda b: tb.solve_Kt1(tb.Mmu @ b))
        return (he, hm, lambda e: tb.K1 @ e, lambda h: tb.Kt1 @ h,
                lambda e: tb.D1 @ e, lambda h: tb.Dt1 @ h)
    from .structured import curl_primal
    return (tb.hodge_eps, tb.hodge_mu,
            lambda e: forms.join(tb.apply_K1(tb.split_e(e))),
            lambda h: forms.join(tb.apply_Kt1(tb.split_h(h))),
            lambda e: forms.join(curl_primal(tb.split_e(e))),
            lambda h: forms.join(curl_dual(tb.split_h(h))))


# ------------------------------------------------------------------------------------------
# BASELINE.json configs[2] (C3) and configs[3] (C4), as SURVEY 8(d) and readings Z16/Z28 define them
# ------------------------------------------------------------------------------------------

C3_SIGMA = 0.05


def c3_setup(p=3, n=48):
    """C3: the map x + 0.1 sin(pi x) sin(pi y) sin(pi z) (1,1,1) interpolated in S_p^3 (reading
    Z18), eps in {1, 4} with the sphere of radius 0.25 at c_eps = rng(3).uniform(.25, .75, 3)
    point-sampled at the physical quadrature points (reading Z17), mu = 1.
    Returns (ctrl, eps at the quadrature points (element-major), physical points [nqp, 3])."""
    from .assemble import Quad, physical_qp
    ctrl = interpolate_map(p, n, c3_map)
    X = physical_qp(Quad(p, forms._n3(n)), ctrl).reshape(-1, 3)
    c_eps, _ = synth.c3_centres()
    eps = np.where(np.linalg.norm(X - c_eps, axis=1) < 0.25, 4.0, 1.0)
    return ctrl, eps, X


def c3_source(p, n, ctrl):
    """C3 source (reading Z16): j^ = D~1 a^ with a^ the unweighted parametric L2 projection onto
    X~1 of A = z-hat exp(-|F(x^) - c_J|^2 / (2 * 0.05^2)) sampled at the physical quadrature points
    (reading Z28), c_J the second rng(3) draw.  Divergence free by D~2 D~1 = 0."""
    _, c_J = synth.c3_centres()
    Xg = physical_points(p, n, ctrl)
    a = project_dual1(p, n, synth.gaussian_z(Xg, c_J, C3_SIGMA))
    tb_n = forms._n3(n)
    return forms.join(curl_dual(forms.split(a, "dual", 1, p, tb_n)))


def c3_amplitudes(dt, n_steps, k0=0):
    """s(t_{k+1/2}) = exp(-((t - 0.15)/0.05)^2) at t = (k + 1/2) dt, k = k0 .. k0 + n_steps - 1."""
    return synth.pulse((np.arange(k0, k0 + n_steps) + 0.5) * dt)


def c4_eps(X):
    """C4: eps = 1 + 0.5 sin(2 pi x) cos(2 pi y) at physical points X[..., 3]."""
    return 1.0 + 0.5 * np.sin(2 * np.pi * X[..., 0]) * np.cos(2 * np.pi * X[..., 1])


def pcg_mass_eps(tb, rhs, tol=1e-14, maxit=500):
    """Solve M~2_{1/eps} d = rhs (tier B, general mass) by preconditioned conjugate gradients with
    the Kronecker preconditioner: the separable mass of the mean 1/eps, inverted mode by mode
    ("d0 by tier-B PCG (Kronecker preconditioner, rel. residual 1e-14)")."""
    from .structured import kron3
    gbar = float(np.mean(tb.inv_eps))
    Binv = [np.linalg.inv(G) for G in tb.GamB1]
    Cinv = [np.linalg.inv(G) for G in tb.GamC2]

    def A(x):
        return forms.join(tb.mass_eps(tb.split_e(x)))

    def Pinv(r):
        rc = tb.split_e(r)
        out = []
        for c in range(3):
            F = [Binv[a] if a == c else Cinv[a] for a in range(3)]
            out.append(kron3(F[0], F[1], F[2], rc[c]) / gbar)
        return forms.join(out)

    x = np.zeros_like(rhs)
    r = rhs.copy()
    z = Pinv(r)
    pv = z.copy()
    rz = r @ z
    nb = np.sqrt(rhs @ rhs)
    for _ in range(maxit):
        q = A(pv)
        al = rz / (pv @ q)
        x += al * pv
        r -= al * q
        if np.sqrt(r @ r) <= tol * nb:
            break
        z = Pinv(r)
        rz_new = r @ z
        pv = z + (rz_new / rz) * pv
        rz = rz_new
    return x


def c4_setup(p=4, n=96):
    """C4: identity map, eps at the quadrature points, mu = 1.  Returns (eps (element-major), tier B)."""
    from .assemble import Quad, physical_qp
    X = physical_qp(Quad(p, forms._n3(n))).reshape(-1, 3)
    eps = c4_eps(X)
    return eps, TierB(p, n, inv_eps=1.0 / eps)


def c4_initial_state(tb, dt):
    """C4: e0 per component = the smoothed N(0,1) draw of rng(4) (synth.smooth_fields),
    d0 = M~2^{-1} K1 e0 by PCG, e0 <- K1^{-1} M~2 d0 (exact consistency), H = 0 so b0 = 0,
    b^{1/2} = -(dt/2) D1 e0 (Taylor half step, reading Z8), h^{1/2} = K~1^{-1} M2 b^{1/2}."""
    from .structured import curl_primal
    shapes = [tuple(s[::-1]) for s in tb.sh_e]  # [z][y][x]
    e0 = forms.join(synth.smooth_fields(4, shapes))
    d0 = pcg_mass_eps(tb, forms.join(tb.apply_K1(tb.split_e(e0))))
    e0 = tb.hodge_eps(d0)
    bh = -0.5 * dt * forms.join(curl_primal(tb.split_e(e0)))
    return d0, e0, bh, tb.hodge_mu(bh)


# ------------------------------------------------------------------------------------------
# consistent initial state
# ------------------------------------------------------------------------------------------

def consistent_state(tb: TierB, d0, bhalf):
    """e0 = K1^{-1} M~2 d0, h^{1/2} = K~1^{-1} M2 b^{1/2} (eqs. discrete2_hodge_eps/mu)."""
    return d0, tb.hodge_eps(d0), bhalf, tb.hodge_mu(bhalf)


def cavity_initial_state(tb: TierB, mode, dt):
    """d0 = projection of D(0) = E(0) onto X~2; b^{1/2} = projection of exact B(dt/2) onto
    X2_{h,0} (reading Z8; identity geometry, eps = mu = 1)."""
    p, n = tb.p, tb.n
    _, _, X = qp_grid(p, n, tb.Q)
    d0 = project_dual2(p, n, mode.E(X, 0.0), tb.Q)
    bh = project_primal2(p, n, mode.B(X, 0.5 * dt), tb.Q)
    return consistent_state(tb, d0, bh)
