"""Pins of the oracle's scheme-2 step (tier A and tier B).

Paper facts: Hodge definition K1 e = M~2 d; Kronecker inverse equals a
dense solve of the assembled block; energy identity eq. energy_aux;
conservation (reading Z5/Z19 for the discrete invariant); Gauss laws;
convergence E ~ h^p, H ~ h^(p-1); first cube mode with energy 1/8 (Z11).
"""
import numpy as np
import pytest

import synth
from oracle import forms
from oracle import workloads as W
from oracle.assemble import Quad, physical_qp
from oracle.scheme import TierA
from oracle.structured import TierB
from conftest import rel


def _rand_state(N_e, N_h, seed):
    g = np.random.default_rng(seed)
    return g.standard_normal(N_e), g.standard_normal(N_e), g.standard_normal(N_h), g.standard_normal(N_h)


@pytest.mark.parametrize("p,n", [(2, 2), (3, 2), (4, 2)])
def test_kronecker_solve_equals_dense_solve(p, n):
    """<= 1000-DoF grids: tier-A sparse direct and tier-B mode-wise both equal numpy.linalg.solve
    of the assembled 3D block (BJ north_star)."""
    A = TierA(p, n)
    B = TierB(p, n)
    r = np.random.default_rng(5).standard_normal(A.N_e)
    rh = np.random.default_rng(6).standard_normal(A.N_h)
    assert A.N_e <= 1000
    Kd, Ktd = A.K1.toarray(), A.Kt1.toarray()
    xd = np.linalg.solve(Kd, r)
    xdh = np.linalg.solve(Ktd, rh)
    # backward-stable solves agree to O(eps * cond) (cond(K1 blocks) <= ~2e4)
    tol = 20 * np.finfo(float).eps * np.linalg.cond(Kd)
    tolh = 20 * np.finfo(float).eps * np.linalg.cond(Ktd)
    assert rel(A.solve_K1(r), xd) < tol
    assert rel(forms.join(B.solve_K1(B.split_e(r))), xd) < tol
    assert rel(A.solve_Kt1(rh), xdh) < tolh
    assert rel(forms.join(B.solve_Kt1(B.split_h(rh))), xdh) < tolh
    # transposed solves
    assert rel(forms.join(B.solve_K1(B.split_e(r), T=True)), np.linalg.solve(Kd.T, r)) < tol


def _c3_like(p, n, seed=0):
    ctrl = W.interpolate_map(p, n, W.c3_map)
    X = physical_qp(Quad(p, n), ctrl)
    c = np.array([0.4, 0.55, 0.5])
    inv_eps = np.where(np.linalg.norm(X - c, axis=-1) < 0.25, 0.25, 1.0).ravel()
    return ctrl, inv_eps


TOL_AB = {2: 1e-14, 3: 1e-13, 4: 5e-12}   # ~ eps x cond(K blocks), cond from SURVEY A2


@pytest.mark.parametrize("p,n", [(2, 3), (3, 3), (4, 2), (2, (3, 2, 4))])
@pytest.mark.parametrize("geom", ["identity", "curved"])
def test_tier_b_equals_tier_a(p, n, geom):
    if geom == "identity":
        A = TierA(p, n)
        B = TierB(p, n)
    else:
        ctrl, ie = _c3_like(p, n)
        A = TierA(p, n, ctrl=ctrl, inv_eps_qp=ie)
        B = TierB(p, n, ctrl=ctrl, inv_eps=ie, inv_mu=1.0)
    st = _rand_state(A.N_e, A.N_h, 7)
    j = np.random.default_rng(8).standard_normal(A.N_e)
    ra = A.step(*st, 0.013, j, 0.7)
    rb = B.step(*st, 0.013, j, 0.7)
    for x, y in zip(rb, ra):
        assert rel(x, y) < TOL_AB[p]
    assert abs(A.energy(*ra) - B.energy(*rb)) < 1e-12 * abs(A.energy(*ra))
    assert np.allclose(A.gauss(ra[0], ra[2]), B.gauss(rb[0], rb[2]), atol=1e-13)


@pytest.mark.parametrize("p,n", [(2, 3), (3, 2)])
def test_hodge_defining_residual(p, n):
    ctrl, ie = _c3_like(p, n)
    A = TierA(p, n, ctrl=ctrl, inv_eps_qp=ie)
    d = np.random.default_rng(9).standard_normal(A.N_e)
    e = A.solve_K1(A.Meps @ d)
    r = A.Meps @ d
    assert np.linalg.norm(A.K1 @ e - r) / np.linalg.norm(r) < 1e-12


@pytest.mark.parametrize("p,n", [(2, 3), (3, 2)])
def test_skew_identity(p, n):
    """e^T K~2 D~1 h = h^T K2 D1 e for any e, h (eq. energy_aux): with
    K~2 = K1^T and K2 = K~1^T."""
    A = TierA(p, n)
    g = np.random.default_rng(10)
    e, h = g.standard_normal(A.N_e), g.standard_normal(A.N_h)
    lhs = e @ (A.K1.T @ (A.Dt1 @ h))
    rhs = h @ (A.Kt1.T @ (A.D1 @ e))
    assert abs(lhs - rhs) < 1e-13 * (abs(lhs) + 1)


def _modified_energy(A, d, e, b_prev, h):
    """E^n = 1/2 d^T K1 e + 1/2 b^{n-1/2 T} K~1 h^{n+1/2}  (reading Z19: exactly invariant)."""
    return 0.5 * d @ (A.K1 @ e) + 0.5 * b_prev @ (A.Kt1 @ h)


def test_modified_energy_exactly_conserved_and_gauss():
    p, n = 3, 2
    ctrl, ie = _c3_like(p, n)
    A = TierA(p, n, ctrl=ctrl, inv_eps_qp=ie)
    B = TierB(p, n, ctrl=ctrl, inv_eps=ie, inv_mu=1.0)
    d, _, b, _ = _rand_state(A.N_e, A.N_h, 11)
    dtmax = W.cfl_dt_max(B)
    dt = 0.9 * dtmax
    e = A.solve_K1(A.Meps @ d)
    h = A.solve_Kt1(A.Mmu @ b)
    g0 = (A.Dt2 @ d, A.D2 @ b)
    Es = []
    b_prev = b
    for k in range(300):
        b_prev = b
        d, e, b, h = A.step(d, e, b, h, dt)
        Es.append(_modified_energy(A, d, e, b_prev, h))
    Es = np.array(Es)
    assert (Es.max() - Es.min()) / abs(Es.mean()) < 1e-13
    # Gauss laws are preserved exactly up to round-off
    assert np.abs(A.Dt2 @ d - g0[0]).max() < 1e-11
    assert np.abs(A.D2 @ b - g0[1]).max() < 1e-11


def test_unstable_above_cfl():
    """Sharpness of the computed stability limit: 1.05 dt_max blows up, 0.95 dt_max stays bounded."""
    p, n = 2, 3
    B = TierB(p, n)
    dtmax = W.cfl_dt_max(B)
    d, _, b, _ = _rand_state(B.N_e, B.N_h, 12)
    out = {}
    for f in (0.95, 1.05):
        x = (d, B.hodge_eps(d), b, B.hodge_mu(b))
        with np.errstate(all="ignore"):
            x = B.run(*x, f * dtmax, 2000)
            nrm = np.linalg.norm(x[0])
        out[f] = nrm if np.isfinite(nrm) else np.inf
    assert out[0.95] < 10 * np.linalg.norm(d)
    assert out[1.05] > 1e3 * np.linalg.norm(d)


def test_poynting_identity_with_divergence_free_source():
    """With j = D~1 a (so D~2 j = 0): E^{n+1} - E^n = -(dt/2)(e^{n+1}+e^n)^T K1^T j^{n+1/2}
    (derived from eq. energy_aux), and Gauss for d is untouched by the source."""
    p, n = 3, 2
    A = TierA(p, n)
    g = np.random.default_rng(13)
    a = g.standard_normal(A.N_h)
    j = A.Dt1 @ a
    assert np.abs(A.Dt2 @ j).max() < 1e-13
    d, _, b, _ = _rand_state(A.N_e, A.N_h, 14)
    e = A.solve_K1(A.Meps @ d)
    h = A.solve_Kt1(A.Mmu @ b)
    dt = 0.01
    E_old = None
    g0 = A.Dt2 @ d
    for k in range(50):
        s = np.sin(0.3 * k)
        e_old, bm = e, b
        d, e, b, h = A.step(d, e, b, h, dt, j, s)
        E_new = _modified_energy(A, d, e, bm, h)
        if E_old is not None:
            pred = -(dt / 2) * (e + e_old) @ (A.K1.T @ (s * j))
            assert abs((E_new - E_old) - pred) < 1e-12 * abs(E_new)
        E_old = E_new
    assert np.abs(A.Dt2 @ d - g0).max() < 1e-11


def test_time_reversibility():
    """Leapfrog is time reversible: undo b then d with the same dt."""
    p, n = 2, 3
    A = TierA(p, n)
    d0, _, b0, _ = _rand_state(A.N_e, A.N_h, 15)
    e0 = A.solve_K1(A.Meps @ d0)
    h0 = A.solve_Kt1(A.Mmu @ b0)
    dt = 0.02
    d, e, b, h = A.run(d0, e0, b0, h0, dt, 30)
    for _ in range(30):
        b = b + dt * (A.D1 @ e)
        h = A.solve_Kt1(A.Mmu @ b)
        d = d - dt * (A.Dt1 @ h)
        e = A.solve_K1(A.Meps @ d)
    assert rel(d, d0) < 1e-12 and rel(b, b0) < 1e-12


def test_first_cube_mode_energy_and_convergence_rates():
    """Cube cavity, first mode (Z11), small fixed dt (reading Z22): relative L2 errors of E and H
    at T decay with rates >= p and >= p-1 (Fig. 2) and the discrete energy tends to the
    exact 1/8."""
    mode = W.CavityMode((1, 1, 0), (0, 0, 1))
    dt, T = 2e-3, 0.2
    ns = int(round(T / dt))
    for p in (2, 3):
        errs, ens = [], []
        for n in (2, 4, 8):
            tb = TierB(p, n)
            st = W.cavity_initial_state(tb, mode, dt)
            ens.append(abs(st[0] @ forms.join(tb.mass_eps(tb.split_e(st[0]))) - 0.25))
            d, e, b, h = tb.run(*st, dt, ns)
            _, _, X = W.qp_grid(p, n)
            errs.append((W.l2_rel_error(p, n, "primal", 1, e, mode.E(X, T)),
                         W.l2_rel_error(p, n, "dual", 1, h, mode.B(X, T + dt / 2))))
        errs = np.array(errs)
        rates = np.log2(errs[:-1] / errs[1:])
        assert rates[-1, 0] > p - 0.3, rates
        assert rates[-1, 1] > p - 1 - 0.3, rates
        # d^T M~2 d with d = projection of E(0) -> int |E|^2 = 1/4 (energy 1/8, eps = 1),
        # with the error of a degree-(p-1)/(p-2) projection: O(h^(2(p-1)))
        ens = np.array(ens)
        assert np.all(np.log2(ens[:-1] / ens[1:]) > 2 * (p - 1) - 0.3), ens
    tb = TierB(3, 8)
    st = W.cavity_initial_state(tb, mode, dt)
    assert abs(tb.energy(*st) - 0.125) < 1e-3


def test_projection_reproduces_members():
    p, n = 3, 3
    tb = TierB(p, n)
    g = np.random.default_rng(16)
    v = g.standard_normal(tb.N_e)
    f = W.eval_form(p, n, "dual", 2, v)
    assert rel(W.project_dual2(p, n, f), v) < 1e-12
    vb = g.standard_normal(tb.N_h)
    fb = W.eval_form(p, n, "primal", 2, vb)
    assert rel(W.project_primal2(p, n, fb), vb) < 1e-12


def test_cfl_scalings():
    """CFL is linear in h (Fig. 5 right) and decreases roughly like 1/p^2 (Fig. 5 left).
    The absolute value is parity-unpinned (reading Z15)."""
    c = {}
    for p, n in ((2, 4), (2, 8), (3, 8), (4, 8)):
        c[(p, n)] = W.cfl_dt_max(TierB(p, n)) * n
    assert abs(c[(2, 4)] / c[(2, 8)] - 1) < 0.05
    slope = np.log(c[(4, 8)] / c[(2, 8)]) / np.log(2.0)
    assert -2.4 < slope < -1.2, slope


def _dense_lambda_max(A):
    """Brute force: the largest eigenvalue of the generalized symmetric problem
    (C^T M2 C) v = lam M~2 v, C = D1 K1^{-1} M~2, from dense assembled tier-A matrices (LAPACK)."""
    import scipy.linalg as sl
    Meps = A.Meps.toarray()
    C = A.D1.toarray() @ np.linalg.solve(A.K1.toarray(), Meps)
    return sl.eigh(C.T @ A.Mmu.toarray() @ C, Meps, eigvals_only=True)[-1]


@pytest.mark.parametrize("case", ["cube_p2", "aniso_p2", "curved_p3"])
def test_cfl_power_pins(case):
    """cfl_power: the Rayleigh quotients are nondecreasing and bounded by the
    brute-force lambda_max (A is M~2-self-adjoint PSD), converge to it, and tier B iterates the same."""
    if case == "cube_p2":
        p, n, kw = 2, 3, {}
    elif case == "aniso_p2":
        p, n, kw = 2, (4, 5, 3), {}
    else:
        p, n = 2, (2, 3, 2)
        ctrl, ie = _c3_like(p, n)
        kw = dict(ctrl=ctrl, inv_eps_qp=ie)
    A = TierA(p, n, **kw)
    lam_d = _dense_lambda_max(A)
    x0 = synth.rng(100).standard_normal(A.N_e)
    iters = 3000 if case == "curved_p3" else 400   # smaller spectral gap on the curved map
    lam, dt, x, lams = W.cfl_power(A, x0, iters)
    lams = np.array(lams)
    assert np.all(np.diff(lams) >= -1e-13 * lam_d)
    assert lams.max() <= lam_d * (1 + 1e-12)
    assert abs(lam / lam_d - 1) < 1e-6, (lam, lam_d)
    assert dt == 2.0 / np.sqrt(lam)
    if case != "curved_p3":
        lamB, _, xB, _ = W.cfl_power(TierB(p, n), x0, 400)
        assert abs(lamB / lam - 1) < 1e-12 and np.abs(xB - x).max() < 1e-10
    else:
        lamB, _, xB, _ = W.cfl_power(TierB(p, n, ctrl=kw["ctrl"], inv_eps=kw["inv_eps_qp"]), x0, iters)
        assert abs(lamB / lam - 1) < 1e-11 and np.abs(xB - x).max() < 1e-8


def test_cfl_p2_closed_form():
    """Derived fact (DESIGN.md readings): on the identity cube with eps = mu = 1 and p = 2,
    lambda_max = (72/5) (n_x^2 + n_y^2 + n_z^2) exactly; checked by dense brute force."""
    for n in (2, 4, (4, 5, 3)):
        nn = np.array(forms._n3(n), dtype=float)
        assert abs(_dense_lambda_max(TierA(2, n)) / (14.4 * (nn ** 2).sum()) - 1) < 1e-12


def test_composed_w1_is_staggered_leapfrog():
    """compose.run_composed with w = (1,) (velocity Verlet, synchronous b) equals the paper's
    staggered leapfrog started from b^{1/2} = b^0 - dt/2 D1 e^0 and read back with
    b^n = b^{n+1/2} + dt/2 D1 e^n."""
    from oracle import compose
    p, n = 3, (3, 2, 4)
    A = TierA(p, n)
    d, _, b, _ = _rand_state(A.N_e, A.N_h, 21)
    e = A.solve_K1(A.Meps @ d)
    h = A.solve_Kt1(A.Mmu @ b)
    dt, steps = 0.01, 7
    out = compose.run_composed(A, d, e, b, h, dt, steps, weights=(1.0,))
    bh = b - 0.5 * dt * (A.D1 @ e)
    st = A.run(d, e, bh, A.solve_Kt1(A.Mmu @ bh), dt, steps)
    bn = st[2] + 0.5 * dt * (A.D1 @ st[1])
    assert rel(out[0], st[0]) < 1e-13 and rel(out[1], st[1]) < 1e-13
    assert rel(out[2], bn) < 1e-13 and rel(out[3], A.solve_Kt1(A.Mmu @ bn)) < 1e-13


@pytest.mark.parametrize("weights,order", [("yoshida", 4), ("verlet", 2)])
def test_composed_time_order_vs_exact_semidiscrete(weights, order):
    """Time order of the composition against the exact solution of the semi-discrete system
    d' = D~1 h, b' = -D1 e (e = K1^{-1} M~2 d, h = K~1^{-1} M2 b; P:L355-372 before the leapfrog),
    y(T) = expm(T L) y(0) from the dense tier-A operator: halving dt divides the error by 2^order."""
    import scipy.linalg as sl
    from oracle import compose
    w = compose.YOSHIDA4 if weights == "yoshida" else (1.0,)
    p, n = 2, 2
    A = TierA(p, n)
    He = np.linalg.solve(A.K1.toarray(), A.Meps.toarray())
    Hm = np.linalg.solve(A.Kt1.toarray(), A.Mmu.toarray())
    Ne, Nh = A.N_e, A.N_h
    L = np.zeros((Ne + Nh, Ne + Nh))
    L[:Ne, Ne:] = A.Dt1.toarray() @ Hm
    L[Ne:, :Ne] = -A.D1.toarray() @ He
    d, _, b, _ = _rand_state(Ne, Nh, 22)
    T = 0.2
    yT = sl.expm(T * L) @ np.concatenate([d, b])
    errs = []
    for m in (16, 32, 64):
        out = compose.run_composed(A, d, He @ d, b, Hm @ b, T / m, m, weights=w)
        errs.append(np.linalg.norm(np.concatenate([out[0], out[2]]) - yT) / np.linalg.norm(yT))
    rates = np.log2(np.array(errs[:-1]) / np.array(errs[1:]))
    assert np.all(np.abs(rates - order) < 0.15), (errs, rates)


# ---- rational (NURBS) maps: the quarter annulus of the coaxial-cable experiment (NEXT #2) ----

def _bernstein_quarter_circle(t):
    """The single-segment rational quadratic quarter circle (control points (1,0), (1,1), (0,1),
    weights 1, 1/sqrt2, 1) evaluated directly in Bernstein form."""
    B = np.stack([(1 - t) ** 2, 2 * t * (1 - t), t ** 2], -1)
    w = np.array([1.0, 1.0 / np.sqrt(2.0), 1.0])
    P = np.array([[1.0, 0.0], [1.0, 1.0], [0.0, 1.0]])
    return (B * w) @ P / (B @ w)[..., None]


@pytest.mark.parametrize("n", [1, (2, 3, 2), (1, 5, 1)])
def test_quarter_annulus_is_exact(n):
    """The NURBS quarter annulus maps onto exact circles r = r1 + (r2 - r1) x^ (closed form), its
    angle follows the single-segment circle after knot insertion (pins Boehm insertion), z is affine."""
    from oracle.workloads import qp_grid
    g = W.quarter_annulus(n, r1=0.5, r2=1.0, height=1.0)
    X = W.physical_points(2, n, g)
    _, _, Xg = qp_grid(2, n, 3)
    r = np.hypot(X[..., 0], X[..., 1])
    assert np.abs(r - (0.5 + 0.5 * Xg[..., 0])).max() < 1e-14
    assert np.abs(X[..., 2] - Xg[..., 2]).max() < 1e-14
    C = _bernstein_quarter_circle(Xg[..., 1])
    assert np.abs(X[..., :2] / r[..., None] - C).max() < 1e-14


@pytest.mark.parametrize("n", [(2, 3, 2), 2])
def test_rational_map_tier_b_equals_tier_a(n):
    """Tier A (3D quadrature with the quotient-rule Jacobian at every point) and tier B (sum
    factorised) agree on the quarter annulus; det DF > 0; the step conserves the modified energy."""
    p = 2
    g = W.quarter_annulus(n)
    A = TierA(p, n, ctrl=g)
    B = TierB(p, n, ctrl=g)
    from oracle.assemble import geometry_at_qp, Quad as Qd
    _, DF = geometry_at_qp(Qd(p, forms._n3(n)), g)
    assert np.linalg.det(DF).min() > 0
    st = _rand_state(A.N_e, A.N_h, 51)
    ra, rb = A.step(*st, 0.01), B.step(*st, 0.01)
    for x, y in zip(rb, ra):
        assert rel(x, y) < 1e-13
    d, e, b, h = st[0], A.solve_K1(A.Meps @ st[0]), st[2], A.solve_Kt1(A.Mmu @ st[2])
    dt = 0.5 * W.cfl_dt_max(B)
    Es = []
    for _ in range(100):
        bp = b
        d, e, b, h = A.step(d, e, b, h, dt)
        Es.append(0.5 * d @ (A.K1 @ e) + 0.5 * bp @ (A.Kt1 @ h))
    assert (max(Es) - min(Es)) / abs(np.mean(Es)) < 1e-12


# ---- the first scheme (mass-matrix Hodge stars) ----

@pytest.mark.parametrize("p,n,tol", [(2, 3, 1e-14), (3, (3, 2, 4), 1e-12), (4, 2, 5e-11)])
def test_scheme1_tier_b_equals_tier_a(p, n, tol):
    """Tier A (assembled 1-form masses M^1_eps, M~^1_mu, SuperLU; eqs. discrete1_*) and tier B
    (Kronecker Grams, dense 1D inverses) agree; tolerance ~ eps x cond of the 1D Grams."""
    from oracle.scheme import TierA1
    from oracle.structured import TierB1
    A, B = TierA1(p, n), TierB1(p, n)
    st = _rand_state(A.N_e, A.N_h, 71)
    j = np.random.default_rng(72).standard_normal(A.N_e)
    for x, y in zip(B.step(*st, 0.01, j, 0.6), A.step(*st, 0.01, j, 0.6)):
        assert rel(x, y) < tol


def test_mass1_affine_scaling():
    """For F(x) = diag(L) x the 1-form mass pulls back with DF^{-1} DF^{-T} det DF = diag(L)^{-2} prod L:
    block c of M^1 equals prod(L) / L_c^2 times the identity-geometry block (closed form)."""
    from oracle.assemble import mass1, Quad as Qd, identity_ctrl
    p, n = 2, (2, 3, 2)
    L = np.array([2.0, 0.5, 1.5])
    q = Qd(p, n)
    M0 = mass1(q, "primal").toarray()
    ML = mass1(q, "primal", ctrl=identity_ctrl(p, n) * L).toarray()
    off = forms.offsets("primal", 1, p, n)
    for c in range(3):
        s = slice(off[c], off[c + 1])
        assert np.abs(ML[s, s] - np.prod(L) / L[c] ** 2 * M0[s, s]).max() < 1e-14 * np.abs(M0[s, s]).max()


def test_scheme1_energy_and_better_cfl():
    """Scheme 1 conserves the modified energy 1/2 d.K1 e + 1/2 b^{n-1/2}.K~1 h^{n+1/2} (its energy
    e.M^1 e = d.K1 e) and has the larger stable step (O(1/p^{3/2}) against
    O(1/p^2) for scheme 2): dense leapfrog-operator spectra on a tiny grid."""
    import scipy.linalg as sl
    from oracle.scheme import TierA1
    ratios = []
    for p in (2, 3, 4):
        A1, A = TierA1(p, 3), TierA(p, 3)
        D1, Dt1 = A1.D1.toarray(), A1.Dt1.toarray()
        H1e = np.linalg.solve(A1.M1eps.toarray(), A1.K1.T.toarray())
        H1m = np.linalg.solve(A1.M1mu.toarray(), A1.Kt1.T.toarray())
        H2e = np.linalg.solve(A.K1.toarray(), A.Meps.toarray())
        H2m = np.linalg.solve(A.Kt1.toarray(), A.Mmu.toarray())
        l1 = np.linalg.eigvals(Dt1 @ H1m @ D1 @ H1e).real.max()
        l2 = np.linalg.eigvals(Dt1 @ H2m @ D1 @ H2e).real.max()
        ratios.append(np.sqrt(l2 / l1))
        if p == 3:
            d, _, b, _ = _rand_state(A1.N_e, A1.N_h, 73)
            e, h = A1.hodge_eps(d), A1.hodge_mu(b)
            Es = []
            for _ in range(200):
                bp = b
                d, e, b, h = A1.step(d, e, b, h, 0.9 * 2 / np.sqrt(l1))
                Es.append(0.5 * d @ (A1.K1 @ e) + 0.5 * bp @ (A1.Kt1 @ h))
            assert (max(Es) - min(Es)) / abs(np.mean(Es)) < 1e-13
    assert ratios[0] > 1 and ratios[1] > ratios[0] and ratios[2] > ratios[1], ratios


@pytest.mark.parametrize("p,n", [(2, 4), (3, (3, 4, 5))])
def test_eh_state_step_equals_four_vector_step(p, n):
    """The (e,h)-state form advances e = K1^{-1} M~2 d and h = K~1^{-1} M2 b exactly as the
    four-vector scheme does: 50 steps with a divergence-free source agree to rounding
    (the four-vector step is pinned by the energy, Gauss and convergence tests above)."""
    from oracle.structured import TierB, curl_dual
    tb = TierB(p, n)
    g = np.random.default_rng(91)
    d, b = g.standard_normal(tb.N_e), g.standard_normal(tb.N_h)
    e, h = tb.hodge_eps(d), tb.hodge_mu(b)
    j = forms.join(curl_dual(tb.split_h(g.standard_normal(tb.N_h))))
    s = np.cos(0.1 * np.arange(50))
    dt = 0.5 * W.cfl_dt_max(tb)
    _, e4, _, h4 = tb.run(d, e, b, h, dt, 50, j, s)
    e2, h2 = tb.run_eh(e, h, dt, 50, j, s)
    assert rel(e2, e4) < 1e-12 and rel(h2, h4) < 1e-12
