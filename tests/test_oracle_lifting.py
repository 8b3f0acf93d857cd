"""Oracle pins of the inhomogeneous Dirichlet lifting and the coaxial-cable TEM workload
(P:L837-849): the lifted scheme converges to the exact standing TEM mode with the paper's rates
(E ~ h^p, H ~ h^{p-1}), reduces to the homogeneous scheme for zero data, conserves the
discrete Gauss law, and its precomputed time-separable vectors reproduce the literal formulation."""
import numpy as np
import pytest

from oracle import forms
from oracle import lifting as Lf
from oracle.scheme import TierA
from conftest import rel


def _errors(p, n, dt, T):
    A, st, g = Lf.coax_setup(p, n, dt)
    K = int(round(T / dt))
    d, e0, bF, h = A.run(*st, dt, K, g)
    eF = g(T) * A.e_hat_b
    eF[A.e_int] = e0
    eE = Lf.l2_error_1form(p, n, A.ctrl, "primalF", eF, lambda X: Lf.tem_E(X, T))
    eH = Lf.l2_error_1form(p, n, A.ctrl, "dual", h, lambda X: Lf.tem_B(X, T + 0.5 * dt))
    return eE, eH


def test_tem_mode_is_an_exact_solution():
    """The standing TEM mode solves Maxwell (eps = mu = 1) in the coax: dE/dt = curl H, dB/dt = -curl E
    by central differences at random points, and E is tangential-free on the cylinders (PEC)."""
    g = np.random.default_rng(3)
    r = g.uniform(Lf.R1, Lf.R2, 20)
    th = g.uniform(0, np.pi / 2, 20)
    X = np.stack([r * np.cos(th), r * np.sin(th), g.uniform(0, 1, 20)], -1)
    t, h = 0.37, 1e-5

    def curl(f, X, t):
        J = np.zeros(X.shape[:-1] + (3, 3))
        for j in range(3):
            dX = np.zeros(3)
            dX[j] = h
            J[..., :, j] = (f(X + dX, t) - f(X - dX, t)) / (2 * h)
        return np.stack([J[..., 2, 1] - J[..., 1, 2], J[..., 0, 2] - J[..., 2, 0], J[..., 1, 0] - J[..., 0, 1]], -1)

    dE = (Lf.tem_E(X, t + h) - Lf.tem_E(X, t - h)) / (2 * h)
    dB = (Lf.tem_B(X, t + h) - Lf.tem_B(X, t - h)) / (2 * h)
    assert np.abs(dE - curl(Lf.tem_B, X, t)).max() < 1e-7
    assert np.abs(dB + curl(Lf.tem_E, X, t)).max() < 1e-7
    for rr in (Lf.R1, Lf.R2):   # E is radial: no tangential part on the cylinders
        Xc = np.stack([rr * np.cos(th), rr * np.sin(th), X[:, 2]], -1)
        E = Lf.tem_E(Xc, t)
        tang = E - (np.sum(E * Xc, -1) / rr ** 2)[:, None] * Xc * np.array([1, 1, 0])
        assert np.abs(tang).max() < 1e-14


def test_coax_tem_convergence_rates():
    """p = 2 (the NURBS degree of the coax map): relative L2 errors at T = 0.3 (dt = 2e-3 fixed, below
    the time-discretisation plateau) fall like h^2 for E and at least like h for H."""
    p, dt, T = 2, 2e-3, 0.3
    errs = [_errors(p, n, dt, T) for n in (2, 4, 8)]
    rE = [np.log2(errs[i][0] / errs[i + 1][0]) for i in range(2)]
    rH = [np.log2(errs[i][1] / errs[i + 1][1]) for i in range(2)]
    assert errs[-1][0] < 0.02 and all(1.7 < r < 2.7 for r in rE), (errs, rE)
    assert errs[-1][1] < 0.03 and all(0.9 < r < 2.3 for r in rH), (errs, rH)


def test_lifting_with_zero_data_is_the_homogeneous_scheme():
    """With e^_b = 0 the lifted tier A (full X^2_h, rectangular D1 and M2) equals tier A on the
    interior vectors, and its boundary b entries stay at their initial values."""
    p, n = 2, (2, 3, 2)
    ctrl = Lf.coax_geometry(n)
    A0 = TierA(p, n, ctrl=ctrl)
    AL = Lf.TierAL(p, n, ctrl, np.zeros(AL_size(p, n)))
    g = np.random.default_rng(5)
    d, b0 = g.standard_normal(A0.N_e), g.standard_normal(A0.N_h)
    bF = np.zeros(AL.N_bF)
    bF[AL.b_int] = b0
    bF[~AL.b_int] = g.standard_normal(int((~AL.b_int).sum())) * 0  # zero boundary flux
    st = (d, A0.solve_K1(A0.Meps @ d), b0, A0.solve_Kt1(A0.Mmu @ b0))
    stL = (d, st[1], bF, st[3])
    for _ in range(5):
        st = A0.step(*st, 0.01)
        stL = AL.step(*stL, 0.01, 0.0)
    assert rel(stL[0], st[0]) < 1e-13 and rel(stL[1], st[1]) < 1e-13 and rel(stL[3], st[3]) < 1e-13
    assert rel(stL[2][AL.b_int], st[2]) < 1e-13 and np.abs(stL[2][~AL.b_int]).max() == 0.0


def AL_size(p, n):
    return forms.form_dim("primalF", 1, p, n)


def test_lifted_step_gauss_law_and_precomputed_vectors():
    """The discrete Gauss laws hold for the lifted scheme (D~2 d and the full D2 b constant),
    and the time-separable precomputation (sgm_step_lifted's w_e, c_b, q0, q1, beta) reproduces the
    literal formulation step by step."""
    p, n, dt = 2, (3, 4, 2), 2e-3
    A, st, g = Lf.coax_setup(p, n, dt)
    V = Lf.lifting_vectors(A, st[2], dt)
    D2F = forms.incidence("primalF", 2, p, A.n)
    gd0, gb0 = A.Dt2 @ st[0], D2F @ st[2]
    d, e0, bF, h = st
    d2, e2, b2, h2 = st[0], st[1], st[2][A.b_int], st[3]
    beta = 0.0
    for k in range(30):
        gk = g((k + 1) * dt)
        d, e0, bF, h = A.step(d, e0, bF, h, dt, gk)
        beta -= dt * gk
        d2 = d2 + dt * (A.Dt1 @ h2)
        e2 = A.solve_K1(A.Meps @ d2) - gk * V["w_e"]
        b2 = b2 - dt * (A.D1 @ e2 + gk * V["c_b"])
        h2 = A.solve_Kt1(A.Mmu @ b2) + V["q0"] + beta * V["q1"]
    assert np.abs(A.Dt2 @ d - gd0).max() < 1e-12 and np.abs(D2F @ bF - gb0).max() < 1e-12
    for x, y in ((d2, d), (e2, e0), (b2, bF[A.b_int]), (h2, h)):
        assert rel(x, y) < 1e-12
