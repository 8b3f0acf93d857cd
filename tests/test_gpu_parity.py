"""GPU parity: the CUDA path through the C ABI against the CPU oracle, element by element on the
same seeded inputs.  Tolerances (north_star / DESIGN.md): relative L2 per vector <= 1e-11 after one
step and <= 1e-9 after 100 steps; standalone kernels <= min(1e-11, 20 eps cond) where cond is the
condition number bound of the Kronecker block (product of the 1D condition numbers); integer
stencils (curls) bit-exact."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2302_04979_b200 as S  # noqa: E402
import synth  # noqa: E402
from oracle import forms  # noqa: E402
from oracle import workloads as W  # noqa: E402
from oracle.structured import TierB, curl_primal, curl_dual  # noqa: E402
from conftest import rel  # noqa: E402

EPS = np.finfo(float).eps


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).cuda()


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


def kron_cond(tb):
    cg = max(np.linalg.cond(G) for G in tb.G)
    cm = max(np.linalg.cond(M) for M in tb.M)
    return max(cg, cm) ** 3


def solve_tol(tb):
    return min(1e-11, 20 * EPS * kron_cond(tb))


SMALL = [(2, 5), (3, (9, 7, 6)), (4, 6), (2, (1, 2, 3))]
MEDIUM = [(3, 32), (2, 64), (4, 33)]


@pytest.mark.parametrize("p,n", SMALL + MEDIUM)
def test_kron_solve(p, n):
    pl = S.Plan(n, p)
    tb = TierB(p, n)
    g = np.random.default_rng(5)
    for which, N, split, solve in ((S.K1, tb.N_e, tb.split_e, tb.solve_K1), (S.KT1, tb.N_h, tb.split_h, tb.solve_Kt1)):
        for T in (False, True):
            r = g.standard_normal(N)
            x = torch.empty(N, dtype=torch.float64, device="cuda")
            pl.kron_solve(which, dev(r), x, transpose=T)
            ref = forms.join(solve(split(r), T=T))
            assert rel(host(x), ref) < solve_tol(tb), (which, T)
            # in place (rhs == x)
            xr = dev(r)
            pl.kron_solve(which, xr, xr, transpose=T)
            assert rel(host(xr), ref) < solve_tol(tb)


@pytest.mark.parametrize("p,n", SMALL + [(3, 20)])
def test_curls_bit_exact(p, n):
    pl = S.Plan(n, p)
    tb = TierB(p, n)
    g = np.random.default_rng(6)
    e = g.standard_normal(tb.N_e)
    h = g.standard_normal(tb.N_h)
    y = torch.empty(tb.N_h, dtype=torch.float64, device="cuda")
    pl.curl(S.CURL_PRIMAL, dev(e), y)
    assert np.array_equal(host(y), forms.join(curl_primal(tb.split_e(e))))
    y2 = torch.empty(tb.N_e, dtype=torch.float64, device="cuda")
    pl.curl(S.CURL_DUAL, dev(h), y2)
    assert np.array_equal(host(y2), forms.join(curl_dual(tb.split_h(h))))


@pytest.mark.parametrize("p,n", SMALL + MEDIUM)
def test_pairing_and_mass_apply(p, n):
    pl = S.Plan(n, p)
    tb = TierB(p, n)
    g = np.random.default_rng(7)
    e = g.standard_normal(tb.N_e)
    h = g.standard_normal(tb.N_h)
    for which, v, split, ap in ((S.K1, e, tb.split_e, tb.apply_K1), (S.KT1, h, tb.split_h, tb.apply_Kt1)):
        for T in (False, True):
            y = torch.empty(v.size, dtype=torch.float64, device="cuda")
            pl.pairing_apply(which, dev(v), y, transpose=T)
            assert rel(host(y), forms.join(ap(split(v), T=T))) < 1e-13
    y = torch.empty(tb.N_e, dtype=torch.float64, device="cuda")
    pl.hodge_apply(S.MASS_EPS, dev(e), y)
    assert rel(host(y), forms.join(tb.mass_eps(tb.split_e(e)))) < 1e-13
    y = torch.empty(tb.N_h, dtype=torch.float64, device="cuda")
    pl.hodge_apply(S.MASS_MU, dev(h), y)
    assert rel(host(y), forms.join(tb.mass_mu(tb.split_h(h)))) < 1e-13
    # full discrete Hodge stars (eqs. discrete2_hodge_eps / _mu)
    y = torch.empty(tb.N_e, dtype=torch.float64, device="cuda")
    pl.hodge_star(S.MASS_EPS, dev(e), y)
    assert rel(host(y), tb.hodge_eps(e)) < solve_tol(tb)
    y = torch.empty(tb.N_h, dtype=torch.float64, device="cuda")
    pl.hodge_star(S.MASS_MU, dev(h), y)
    assert rel(host(y), tb.hodge_mu(h)) < solve_tol(tb)


def _state(tb, seed):
    g = np.random.default_rng(seed)
    return g.standard_normal(tb.N_e), g.standard_normal(tb.N_e), g.standard_normal(tb.N_h), g.standard_normal(tb.N_h)


def _run_gpu(pl, st, dt, n_steps, jhat=None, jamp=None):
    d, e, b, h = (dev(x) for x in st)
    pl.step(d, e, b, h, dt, n_steps, j_hat=None if jhat is None else dev(jhat),
            j_amp=None if jamp is None else dev(jamp))
    return [host(x) for x in (d, e, b, h)]


@pytest.mark.parametrize("p,n", SMALL + [(3, 24)])
def test_step_parity_1_and_100(p, n):
    pl = S.Plan(n, p)
    tb = TierB(p, n)
    st = _state(tb, 8)
    dt = 0.4 * W.cfl_dt_max(tb) if tb.N_e < 20000 else 0.1 / max(forms._n3(n))
    out = _run_gpu(pl, st, dt, 1)
    ref = tb.step(*st, dt)
    for a, b in zip(out, ref):
        assert rel(a, b) < 1e-11
    out = _run_gpu(pl, st, dt, 100)
    ref = tb.run(*st, dt, 100)
    for a, b in zip(out, ref):
        assert rel(a, b) < 1e-9


def test_step_with_source_and_amplitudes():
    p, n = 3, (7, 6, 5)
    pl = S.Plan(n, p)
    tb = TierB(p, n)
    st = _state(tb, 9)
    a = np.random.default_rng(10).standard_normal(tb.N_h)
    jhat = forms.join(curl_dual(tb.split_h(a)))        # divergence free
    jamp = np.sin(0.3 * np.arange(40))
    dt = 0.4 * W.cfl_dt_max(tb)
    out = _run_gpu(pl, st, dt, 40, jhat, jamp)
    ref = tb.run(*st, dt, 40, jhat, jamp)
    for x, y in zip(out, ref):
        assert rel(x, y) < 1e-10
    assert pl.check_source(dev(jhat)) == 0
    assert pl.check_source(dev(np.random.default_rng(11).standard_normal(tb.N_e))) == 6


def test_energy_and_gauss():
    p, n = 3, (8, 7, 9)
    pl = S.Plan(n, p)
    tb = TierB(p, n)
    st = _state(tb, 12)
    out = torch.zeros(2, dtype=torch.float64, device="cuda")
    pl.energy(*(dev(x) for x in st), out)
    E = host(out)[0]
    assert abs(E - tb.energy(*st)) < 1e-12 * abs(tb.energy(*st))
    pl.gauss(dev(st[0]), dev(st[2]), out)
    gg = host(out)
    ref = tb.gauss(st[0], st[2])
    assert abs(gg[0] - ref[0]) <= 1e-15 * ref[0] and abs(gg[1] - ref[1]) <= 1e-15 * ref[1]


def _curved_case(p, n, incl=True):
    ctrl = W.interpolate_map(p, n, W.c3_map)
    X = W.physical_points(p, n, ctrl)
    Xel = np.stack([W.grid_to_elem(X[..., i], n, p + 1) for i in range(3)], -1)
    eps = np.where(np.linalg.norm(Xel - np.array([0.45, 0.5, 0.55]), axis=-1) < 0.25, 4.0, 1.0) if incl \
        else np.ones(Xel.shape[0])
    return ctrl, eps


@pytest.mark.parametrize("p,n", [(3, (6, 5, 7)), (2, 6), (4, (5, 4, 4))])
def test_general_hodge_curved_step(p, n):
    ctrl, eps = _curved_case(p, n)
    pl = S.Plan(n, p, geom_ctrl=ctrl)
    pl.set_material(S.EPS, eps)
    assert not pl.separable(S.MASS_EPS) and not pl.separable(S.MASS_MU)
    tb = TierB(p, n, ctrl=ctrl, inv_eps=1.0 / eps, inv_mu=1.0)
    tb.sep_mu = None
    tb.W_mu = tb._W(1.0)
    g = np.random.default_rng(13)
    x = g.standard_normal(tb.N_e)
    y = torch.empty(tb.N_e, dtype=torch.float64, device="cuda")
    pl.hodge_apply(S.MASS_EPS, dev(x), y)
    assert rel(host(y), forms.join(tb.mass_eps(tb.split_e(x)))) < 1e-13
    xb = g.standard_normal(tb.N_h)
    yb = torch.empty(tb.N_h, dtype=torch.float64, device="cuda")
    pl.hodge_apply(S.MASS_MU, dev(xb), yb)
    assert rel(host(yb), forms.join(tb.mass_mu(tb.split_h(xb)))) < 1e-13
    st = _state(tb, 14)
    dt = 0.02 / max(forms._n3(n))
    out = _run_gpu(pl, st, dt, 1)
    for a, b in zip(out, tb.step(*st, dt)):
        assert rel(a, b) < 1e-11
    out = _run_gpu(pl, st, dt, 20)
    for a, b in zip(out, tb.run(*st, dt, 20)):
        assert rel(a, b) < 1e-10


def test_general_hodge_variable_eps_identity():
    p, n = 4, 6
    pl = S.Plan(n, p)
    X = pl.qp_coords()
    eps = 1 + 0.5 * np.sin(2 * np.pi * X[:, 0]) * np.cos(2 * np.pi * X[:, 1])
    pl.set_material(S.EPS, eps)
    assert not pl.separable(S.MASS_EPS) and pl.separable(S.MASS_MU)
    tb = TierB(p, n, inv_eps=1.0 / eps)
    st = _state(tb, 15)
    dt = 0.01
    out = _run_gpu(pl, st, dt, 1)
    for a, b in zip(out, tb.step(*st, dt)):
        assert rel(a, b) < 1e-11


@pytest.mark.parametrize("p,axis,curved", [(4, 0, False), (4, 2, False), (3, 1, True), (3, 2, True), (2, 0, True)])
def test_general_hodge_long_axis_uniform_bricks(p, axis, curved):
    """100 elements along one axis (5 and 6 along the others: ragged bricks): most bricks / layers
    along the long axis are interior, so the brick kernel reads their element tables from its
    parameters (the host makes the interior tables bit-identical: at n ~ 100 their construction
    rounding, n * 1e-16, is above the 1e-14 the kernel used to test with), W comes from the
    brick-layout chunks, and along z the chunking is the cost-based one.  Both masses against the
    oracle's mass applies (scalar W on the identity map, full W on the curved map)."""
    n = [5, 6, 5]
    n[axis] = 100
    n = tuple(n)
    if curved:
        ctrl, eps = _curved_case(p, n, incl=False)
        pl = S.Plan(n, p, geom_ctrl=ctrl)
        X = pl.qp_coords()
        eps = 1 + 0.4 * np.sin(2 * np.pi * X[:, 0]) * np.cos(2 * np.pi * X[:, 2])
        mu = 1 + 0.3 * np.cos(2 * np.pi * X[:, 1])
        tb = TierB(p, n, ctrl=ctrl, inv_eps=1.0 / eps, inv_mu=1.0 / mu)
    else:
        pl = S.Plan(n, p)
        X = pl.qp_coords()
        eps = 1 + 0.5 * np.sin(2 * np.pi * X[:, 0]) * np.cos(2 * np.pi * X[:, 1])
        mu = 1 + 0.25 * np.sin(2 * np.pi * X[:, 2])
        tb = TierB(p, n, inv_eps=1.0 / eps, inv_mu=1.0 / mu)
    pl.set_material(S.EPS, eps)
    pl.set_material(S.MU, mu)
    assert not pl.separable(S.MASS_EPS) and not pl.separable(S.MASS_MU)
    g = np.random.default_rng(131 + p + axis)
    x = g.standard_normal(tb.N_e)
    y = torch.empty(tb.N_e, dtype=torch.float64, device="cuda")
    pl.hodge_apply(S.MASS_EPS, dev(x), y)
    assert rel(host(y), forms.join(tb.mass_eps(tb.split_e(x)))) < 1e-13
    xb = g.standard_normal(tb.N_h)
    yb = torch.empty(tb.N_h, dtype=torch.float64, device="cuda")
    pl.hodge_apply(S.MASS_MU, dev(xb), yb)
    assert rel(host(yb), forms.join(tb.mass_mu(tb.split_h(xb)))) < 1e-13
    y2 = torch.empty_like(y)
    pl.hodge_apply(S.MASS_EPS, dev(x), y2)
    assert torch.equal(y, y2)


def test_step_host_equals_device():
    p, n = 3, 10
    pl = S.Plan(n, p)
    tb = TierB(p, n)
    st = _state(tb, 16)
    dt = 0.01
    dv = _run_gpu(pl, st, dt, 3)
    hs = [x.copy() for x in st]
    pl.step_host(*hs, dt, 3)
    for a, b in zip(hs, dv):
        assert np.array_equal(a, b)
    # the input e is never read by a step (not even uploaded): NaN in, the same state out
    hs = [x.copy() for x in st]
    hs[1][:] = np.nan
    pl.step_host(*hs, dt, 3)
    for a, b in zip(hs, dv):
        assert np.array_equal(a, b)
    # n_steps = 0: everything round-trips unchanged
    hs = [x.copy() for x in st]
    pl.step_host(*hs, dt, 0)
    for a, b in zip(hs, st):
        assert np.array_equal(a, b)


def test_c1_cavity_vs_tier_a():
    """configs[0]: cube cavity, p = 2, 8^3, first mode, 20 steps at dt = 0.5 CFL; GPU vs the plain
    definition (tier A, SuperLU) and the exact energy 1/8."""
    from oracle.scheme import TierA
    p, n = 2, 8
    tb = TierB(p, n)
    dt = 0.5 * W.cfl_dt_max(tb)
    mode = W.CavityMode((1, 1, 0), (0, 0, 1))
    st = W.cavity_initial_state(tb, mode, dt)
    pl = S.Plan(n, p)
    out = _run_gpu(pl, st, dt, 20)
    A = TierA(p, n)
    ref = A.run(*st, dt, 20)
    for a, b in zip(out, ref):
        assert rel(a, b) < 1e-10
    E = torch.zeros(1, dtype=torch.float64, device="cuda")
    pl.energy(*(dev(x) for x in out), E)
    assert abs(host(E)[0] - 0.125) < 0.01


def test_nan_poisoned_workspace_and_graph_replay():
    """The workspace (inter-sweep temporary and reduction partials) is fully overwritten before it
    is read: poisoning it with NaN changes nothing.  Also: sgm_step on a non-default stream replays a
    captured CUDA graph for identical calls; results equal the oracle both times."""
    p, n = 3, (33, 7, 9)
    pl = S.Plan(n, p)
    tb = TierB(p, n)
    st = _state(tb, 21)
    dt = 0.01
    ws = torch.full(((pl.workspace_bytes() + 7) // 8,), float("nan"), dtype=torch.float64, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        d, e, b, h = (dev(x) for x in st)
        pl.step(d, e, b, h, dt, 2, ws=ws, stream=s)          # captured
        ref = tb.run(*st, dt, 2)
        out = [host(x) for x in (d, e, b, h)]
        for a, r in zip(out, ref):
            assert np.all(np.isfinite(a)) and rel(a, r) < 1e-11
        d2, e2, b2, h2 = (dev(x) for x in st)
        ws.fill_(float("nan"))
        # different pointers -> re-capture; then the same pointers again -> replay
        pl.step(d2, e2, b2, h2, dt, 2, ws=ws, stream=s)
        pl.step(d2, e2, b2, h2, dt, 2, ws=ws, stream=s)
        ref2 = tb.run(*ref, dt, 2)
        for a, r in zip((d2, e2, b2, h2), ref2):
            assert rel(host(a), r) < 1e-11


def test_multi_step_graph_chunks():
    """A long sgm_step call on a non-default stream replays a graph of 8 captured steps (captured
    with the one-step graph at the first call) plus one-step graphs for the remainder: 19 steps
    = 2 chunks + 3 single steps equal direct launches (SGM_OPT_NO_GRAPH) bit for bit and the
    oracle to the step tolerance."""
    p, n = 3, (12, 9, 10)
    pl = S.Plan(n, p)
    tb = TierB(p, n)
    st = _state(tb, 23)
    dt = 0.01
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        a = [dev(x) for x in st]
        pl.step(*a, dt, 1, stream=s)     # first call: captures the one-step and the 8-step graphs
        pl.step(*a, dt, 19, stream=s)    # 2 chunk replays + 3 one-step replays
        pl.set_options(S.OPT_NO_GRAPH)
        bb = [dev(x) for x in st]
        pl.step(*bb, dt, 20, stream=s)   # direct launches
        pl.set_options(0)
    s.synchronize()
    ref = tb.run(*st, dt, 20)
    for x, y, r in zip(a, bb, ref):
        assert torch.equal(x, y)
        assert rel(host(x), r) < 1e-10


def test_gpu_invariants_over_many_steps():
    """Through the GPU path only (no oracle): the scheme-2 invariants hold over 400 steps of a
    16^3 p = 3 cavity with a random state: the modified energy
    E^ = 1/2 d^{n+1}.K1 e^{n+1} + 1/2 b^{n+1/2}.K~1 h^{n+3/2} is constant (reading Z19)
    and the discrete Gauss laws D~2 d, D2 b are preserved."""
    p, n = 3, 16
    pl = S.Plan(n, p)
    tb = TierB(p, n)
    g = np.random.default_rng(30)
    dt = 0.45 * 0.2020 / n
    d, b = dev(g.standard_normal(tb.N_e)), dev(g.standard_normal(tb.N_h))
    e, h = torch.empty_like(d), torch.empty_like(b)
    pl.hodge_star(S.MASS_EPS, d, e)
    pl.hodge_star(S.MASS_MU, b, h)
    out = torch.zeros(2, dtype=torch.float64, device="cuda")
    pl.gauss(d, b, out)
    g0 = host(out).copy()
    K1e, Kt1h = torch.empty_like(d), torch.empty_like(b)
    energies = []
    for _ in range(40):
        pl.step(d, e, b, h, dt, 9)
        b_prev = b.clone()
        pl.step(d, e, b, h, dt, 1)
        pl.pairing_apply(S.K1, e, K1e)
        pl.pairing_apply(S.KT1, h, Kt1h)
        energies.append(0.5 * float(torch.dot(d, K1e)) + 0.5 * float(torch.dot(b_prev, Kt1h)))
    energies = np.array(energies)
    assert np.ptp(energies) < 1e-12 * abs(energies.mean())
    pl.gauss(d, b, out)
    scale = max(float(torch.max(torch.abs(d))), float(torch.max(torch.abs(b))))
    assert np.all(np.abs(host(out) - g0) <= 1e-11 * scale)


def _cfl_gpu(pl, x0, n_iter):
    x = dev(x0)
    e = torch.empty(pl.N_e, dtype=torch.float64, device="cuda")
    b = torch.empty(pl.N_h, dtype=torch.float64, device="cuda")
    h = torch.empty_like(b)
    out = torch.zeros(2, dtype=torch.float64, device="cuda")
    pl.cfl(x, e, b, h, out, n_iter)
    return host(out), host(x)


@pytest.mark.parametrize("case", ["cube_p2", "ragged_p3", "curved_p3", "p4"])
def test_cfl_power_parity(case):
    """sgm_cfl against oracle workloads.cfl_power: same start vector rng(100), same iteration count.
    Power iteration does not amplify rounding, so lambda agrees to 1e-11 and the iterate to 1e-9."""
    ctrl = None
    if case == "cube_p2":
        p, n = 2, 8
    elif case == "ragged_p3":
        p, n = 3, (9, 7, 6)
    elif case == "p4":
        p, n = 4, 6
    else:
        p, n = 3, (6, 5, 7)
        ctrl, eps = _curved_case(p, n)
    pl = S.Plan(n, p, geom_ctrl=ctrl)
    if ctrl is not None:
        pl.set_material(S.EPS, eps)
        tb = TierB(p, n, ctrl=ctrl, inv_eps=1.0 / eps, inv_mu=1.0)
    else:
        tb = TierB(p, n)
    x0 = synth.rng(100).standard_normal(tb.N_e)
    for iters in (1, 60):
        lam, dt, xr, _ = W.cfl_power(tb, x0, iters)
        out, x = _cfl_gpu(pl, x0, iters)
        assert abs(out[0] / lam - 1) < 1e-11 and abs(out[1] / dt - 1) < 1e-11, (iters, out, lam)
        assert np.abs(x - xr).max() < 1e-9
    if case == "cube_p2":   # closed form: lambda_max = 72/5 * 3 n^2, approached from below
        bound = 14.4 * 3 * n * n
        out, _ = _cfl_gpu(pl, x0, 1500)
        assert bound * (1 - 2e-3) < out[0] <= bound * (1 + 1e-12), (out[0], bound)


@pytest.mark.parametrize("case", ["yoshida_src", "verlet", "curved_yoshida", "five_stage"])
def test_step_composed_parity(case):
    """sgm_step_composed against oracle compose.run_composed (unmerged kick-drift-kick sub-steps):
    the GPU merges adjacent half kicks, so the two differ only by rounding."""
    from oracle import compose
    ctrl = None
    p, n = 3, (7, 6, 5)
    w = compose.YOSHIDA4
    if case == "verlet":
        p, n, w = 2, 6, (1.0,)
    elif case == "five_stage":   # Suzuki's 4th-order fractal composition (symmetric, 5 stages)
        z = 1.0 / (4.0 - 4.0 ** (1.0 / 3.0))
        p, n, w = 4, (5, 6, 4), (z, z, 1.0 - 4.0 * z, z, z)
    elif case == "curved_yoshida":
        p, n = 3, (6, 5, 7)
        ctrl, eps = _curved_case(p, n)
    pl = S.Plan(n, p, geom_ctrl=ctrl)
    if ctrl is not None:
        pl.set_material(S.EPS, eps)
        tb = TierB(p, n, ctrl=ctrl, inv_eps=1.0 / eps, inv_mu=1.0)
    else:
        tb = TierB(p, n)
    st = _state(tb, 31)
    jhat = jamp = None
    steps = 12
    if case == "yoshida_src":
        a = np.random.default_rng(32).standard_normal(tb.N_h)
        jhat = forms.join(curl_dual(tb.split_h(a)))
        jamp = np.cos(0.2 * np.arange(steps * len(w)))
    dt = 0.2 * W.cfl_dt_max(tb)
    for k in (1, steps):
        d, e, b, h = (dev(x) for x in st)
        pl.step_composed(d, e, b, h, dt, w, k, j_hat=None if jhat is None else dev(jhat),
                         j_amp=None if jamp is None else dev(jamp[:k * len(w)]))
        ref = compose.run_composed(tb, *st, dt, k, weights=w, jhat=jhat,
                                   jamp=None if jamp is None else jamp[:k * len(w)])
        for x, y in zip((d, e, b, h), ref):
            assert rel(host(x), y) < (1e-11 if k == 1 else 1e-10), (case, k)


SCHEDULES = [0, S.OPT_FULL_SCHEDULE, S.OPT_FUSED, S.OPT_FUSED | S.OPT_FULL_SCHEDULE, S.OPT_SERIAL,
             S.OPT_EXACT_SPIKE, S.OPT_NO_GRAPH, S.OPT_FUSED | S.OPT_EXACT_SPIKE, S.OPT_WIDE_TILES,
             S.OPT_WIDE_TILES | S.OPT_FULL_SCHEDULE | S.OPT_SERIAL]


@pytest.mark.parametrize("opts", SCHEDULES)
@pytest.mark.parametrize("p,n", [(2, (5, 9, 7)), (3, 11), (4, (6, 5, 8))])
def test_reduced_and_full_schedules(p, n, opts):
    """Every schedule option (separate or fused update; reduced: diagonal factors
    as per-line scalings / full: every axis swept; exact or truncated SPIKE; serial; no graph) against
    the oracle: Hodge stars and 30 steps."""
    pl = S.Plan(n, p)
    pl.set_options(opts)
    assert pl.reduced_schedule() == (not opts & S.OPT_FULL_SCHEDULE)
    tb = TierB(p, n)
    g = np.random.default_rng(41)
    x = g.standard_normal(tb.N_e)
    y = torch.empty(tb.N_e, dtype=torch.float64, device="cuda")
    pl.hodge_star(S.MASS_EPS, dev(x), y)
    assert rel(host(y), tb.hodge_eps(x)) < solve_tol(tb)
    xb = g.standard_normal(tb.N_h)
    yb = torch.empty(tb.N_h, dtype=torch.float64, device="cuda")
    pl.hodge_star(S.MASS_MU, dev(xb), yb)
    assert rel(host(yb), tb.hodge_mu(xb)) < solve_tol(tb)
    st = _state(tb, 42)
    dt = 0.4 * W.cfl_dt_max(tb)
    out = _run_gpu(pl, st, dt, 30)
    for a, b in zip(out, tb.run(*st, dt, 30)):
        assert rel(a, b) < 1e-10


def test_graph_replay_with_per_step_amplitude():
    """A simulation loop that refreshes one device scalar s_k and calls sgm_step(n_steps=1, j_amp=s)
    on a non-default stream: the captured step is replayed and reads the current s every step."""
    p, n = 3, (7, 6, 8)
    pl = S.Plan(n, p)
    tb = TierB(p, n)
    st = _state(tb, 23)
    a = np.random.default_rng(24).standard_normal(tb.N_h)
    jhat = forms.join(curl_dual(tb.split_h(a)))
    amps = np.sin(0.4 * np.arange(12)) + 0.5
    dt = 0.3 * W.cfl_dt_max(tb)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        d, e, b, h = (dev(x) for x in st)
        jh = dev(jhat)
        sbuf = torch.empty(1, dtype=torch.float64, device="cuda")
        for k in range(len(amps)):
            sbuf.fill_(float(amps[k]))
            pl.step(d, e, b, h, dt, 1, j_hat=jh, j_amp=sbuf, stream=s)
        out = [host(x) for x in (d, e, b, h)]
    ref = tb.run(*st, dt, len(amps), jhat, amps)
    for x, y in zip(out, ref):
        assert rel(x, y) < 1e-10


@pytest.mark.parametrize("otf", [False, True])
@pytest.mark.parametrize("n", [(6, 7, 5), 8])
def test_rational_quarter_annulus(n, otf):
    """The coaxial-cable cross-section as an exact degree-2 NURBS map (quarter annulus): general
    Hodge applies and 1 / 20 steps against tier B (which evaluates the same rational map itself).
    SGM_OPT_OTF_GEOMETRY does not apply to rational maps: the stored weights are used."""
    p = 2
    g = W.quarter_annulus(n)
    pl = S.Plan(n, p, geom_ctrl=g)
    if otf:
        pl.set_options(S.OPT_OTF_GEOMETRY)
    tb = TierB(p, n, ctrl=g)
    rng = np.random.default_rng(61)
    x = rng.standard_normal(tb.N_e)
    y = torch.empty(tb.N_e, dtype=torch.float64, device="cuda")
    pl.hodge_apply(S.MASS_EPS, dev(x), y)
    assert rel(host(y), forms.join(tb.mass_eps(tb.split_e(x)))) < 1e-13
    xb = rng.standard_normal(tb.N_h)
    yb = torch.empty(tb.N_h, dtype=torch.float64, device="cuda")
    pl.hodge_apply(S.MASS_MU, dev(xb), yb)
    assert rel(host(yb), forms.join(tb.mass_mu(tb.split_h(xb)))) < 1e-13
    st = _state(tb, 62)
    dt = 0.4 * W.cfl_dt_max(tb)
    for k, tol in ((1, 1e-11), (20, 1e-10)):
        out = _run_gpu(pl, st, dt, k)
        for a, b in zip(out, tb.run(*st, dt, k)):
            assert rel(a, b) < tol


@pytest.mark.parametrize("p,n", [(2, (5, 9, 7)), (3, 11), (3, (9, 7, 6)), (4, (6, 7, 5))])
def test_scheme1_parity(p, n):
    """The first scheme (mass-matrix Hodge stars) on the GPU against oracle tier B1:
    the two Hodge stars, 1 and 30 steps, and the power-iteration stability limit."""
    from oracle.structured import TierB1
    pl = S.Plan(n, p)
    pl.set_scheme(1)
    tb = TierB1(p, n)
    rng = np.random.default_rng(81)
    x = rng.standard_normal(tb.N_e)
    y = torch.empty(tb.N_e, dtype=torch.float64, device="cuda")
    pl.hodge_star(S.MASS_EPS, dev(x), y)
    assert rel(host(y), tb.hodge_eps(x)) < 1e-11
    xb = rng.standard_normal(tb.N_h)
    yb = torch.empty(tb.N_h, dtype=torch.float64, device="cuda")
    pl.hodge_star(S.MASS_MU, dev(xb), yb)
    assert rel(host(yb), tb.hodge_mu(xb)) < 1e-11
    x0 = synth.rng(100).standard_normal(tb.N_e)
    lam, dtmax, _, _ = W.cfl_power(tb, x0, 40)
    out, _ = _cfl_gpu(pl, x0, 40)
    assert abs(out[0] / lam - 1) < 1e-10
    st = (x, tb.hodge_eps(x), xb, tb.hodge_mu(xb))
    dt = 0.4 * dtmax
    for k, tol in ((1, 1e-11), (30, 1e-10)):
        o = _run_gpu(pl, st, dt, k)
        for a, b in zip(o, tb.run(*st, dt, k)):
            assert rel(a, b) < tol


def test_scheme1_composed_yoshida():
    """sgm_step_composed with the first scheme's Hodge stars against oracle compose.run_composed
    on tier B1 (the composition only calls the stars and the curls)."""
    from oracle import compose
    from oracle.structured import TierB1
    p, n = 3, (7, 6, 8)
    pl = S.Plan(n, p)
    pl.set_scheme(1)
    tb = TierB1(p, n)
    st = _state(tb, 91)
    dt = 0.2 * W.cfl_dt_max(TierB(p, n))
    d, e, b, h = (dev(x) for x in st)
    pl.step_composed(d, e, b, h, dt, compose.YOSHIDA4, 6)
    ref = compose.run_composed(tb, *st, dt, 6)
    for x, y in zip((d, e, b, h), ref):
        assert rel(host(x), y) < 1e-10


@pytest.mark.parametrize("case", ["var_eps", "curved", "var_eps_p4"])
def test_scheme1_pcg_parity(case):
    """Scheme 1 with non-separable 1-form masses (variable eps on the identity map; the curved C3-type
    map with an eps inclusion): the GPU's preconditioned-CG Hodge stars (separable scheme-1 star as
    preconditioner, fixed 40 iterations) against tier A1's SuperLU solves of the assembled masses,
    then 1 and 10 steps and the stability limit."""
    from oracle.scheme import TierA1
    p = 4 if case == "var_eps_p4" else 3
    if case.startswith("var_eps"):
        n, ctrl = (5, 6, 4), None
        pl = S.Plan(n, p)
        X = pl.qp_coords()
        eps = 1 + 0.5 * np.sin(2 * np.pi * X[:, 0]) * np.cos(2 * np.pi * X[:, 1])
    else:
        n = (4, 5, 4)
        ctrl, eps = _curved_case(p, n)
        pl = S.Plan(n, p, geom_ctrl=ctrl)
    pl.set_material(S.EPS, eps)
    pl.set_scheme(1)
    A = TierA1(p, n, ctrl=ctrl, eps_qp=eps)
    rng = np.random.default_rng(95)
    x = rng.standard_normal(A.N_e)
    y = torch.empty(A.N_e, dtype=torch.float64, device="cuda")
    pl.hodge_star(S.MASS_EPS, dev(x), y)
    assert rel(host(y), A.hodge_eps(x)) < 1e-11
    xb = rng.standard_normal(A.N_h)
    yb = torch.empty(A.N_h, dtype=torch.float64, device="cuda")
    pl.hodge_star(S.MASS_MU, dev(xb), yb)
    assert rel(host(yb), A.hodge_mu(xb)) < 1e-11
    st = (x, A.hodge_eps(x), xb, A.hodge_mu(xb))
    lam, dtmax, _, _ = W.cfl_power(A, synth.rng(100).standard_normal(A.N_e), 30)
    out, _ = _cfl_gpu(pl, synth.rng(100).standard_normal(A.N_e), 30)
    assert abs(out[0] / lam - 1) < 1e-9
    dt = 0.4 * dtmax
    for k, tol in ((1, 1e-11), (10, 1e-10)):
        o = _run_gpu(pl, st, dt, k)
        for a_, b_ in zip(o, A.run(*st, dt, k)):
            assert rel(a_, b_) < tol


@pytest.mark.parametrize("seed", range(6))
def test_random_shapes(seed):
    """Seeded random degrees and anisotropic element counts (including single-element axes and long
    thin boxes that change the sweep tiling, segment counts and fork/merge decisions): Hodge stars
    and 5 steps of both schemes against the oracle."""
    from oracle.structured import TierB1
    g = np.random.default_rng(1000 + seed)
    p = int(g.integers(2, 5))
    n = tuple(int(v) for v in g.choice([1, 2, 3, 5, 8, 13, 21, 34], size=3))
    for scheme in (2, 1):
        pl = S.Plan(n, p)
        if scheme == 1:
            pl.set_scheme(1)
        tb = TierB(p, n) if scheme == 2 else TierB1(p, n)
        st = _state(tb, 2000 + seed)
        x = st[0]
        y = torch.empty(tb.N_e, dtype=torch.float64, device="cuda")
        pl.hodge_star(S.MASS_EPS, dev(x), y)
        assert rel(host(y), tb.hodge_eps(x)) < 1e-11, (p, n, scheme)
        dt = 0.02 / max(n)
        out = _run_gpu(pl, st, dt, 5)
        for a_, b_ in zip(out, tb.run(*st, dt, 5)):
            assert rel(a_, b_) < 1e-10, (p, n, scheme)


def test_step_composed_graph_replay():
    """sgm_step_composed on a non-default stream: the first call captures its launch sequence, later
    identical calls replay it; 8 calls of one Yoshida step equal the oracle's 8 composed steps."""
    from oracle import compose
    p, n = 3, (6, 7, 5)
    pl = S.Plan(n, p)
    tb = TierB(p, n)
    st = _state(tb, 97)
    dt = 0.2 * W.cfl_dt_max(tb)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        d, e, b, h = (dev(x) for x in st)
        for _ in range(8):
            pl.step_composed(d, e, b, h, dt, compose.YOSHIDA4, 1, stream=s)
        out = [host(x) for x in (d, e, b, h)]
    ref = st
    for _ in range(8):
        ref = compose.run_composed(tb, *ref, dt, 1)
    for x, y in zip(out, ref):
        assert rel(x, y) < 1e-10


def test_abi_argument_validation_on_device():
    """Device plans validate before launching (SGM_E_INVALID_ARG = 1, nothing modified): aliasing
    state vectors, a too-small workspace, non-finite dt, negative n_steps, bad composition weights,
    distinctness in sgm_cfl; a non-divergence-free source is reported by sgm_check_source."""
    import ctypes
    p, n = 2, 4
    pl = S.Plan(n, p)
    st = _state(TierB(p, n), 3)
    d, e, b, h = (dev(x) for x in st)
    keep = [host(x) for x in (d, e, b, h)]
    ws = pl.workspace()
    P = S._ptr
    nb = ws.numel() * 8
    assert S.sgm_step(pl.h, P(d), P(d), P(b), P(h), None, None, 0.01, 1, P(ws), nb, None) == 1
    assert S.sgm_step(pl.h, P(d), P(e), P(b), P(h), None, None, 0.01, 1, P(ws), 64, None) == 1
    assert S.sgm_step(pl.h, P(d), P(e), P(b), P(h), None, None, float("nan"), 1, P(ws), nb, None) == 1
    assert S.sgm_step(pl.h, P(d), P(e), P(b), P(h), None, None, 0.01, -1, P(ws), nb, None) == 1
    w = np.array([1.0, float("inf")])
    assert S.sgm_step_composed(pl.h, P(d), P(e), P(b), P(h), None, None, w.ctypes.data, 2, 0.01, 1,
                               P(ws), nb, None) == 1
    out = torch.zeros(2, dtype=torch.float64, device="cuda")
    assert S.sgm_cfl(pl.h, P(d), P(d), P(b), P(h), 3, P(out), P(ws), nb, None) == 1
    for a, k in zip((d, e, b, h), keep):
        assert np.array_equal(host(a), k)
    assert "alias" in S._lib.sgm_last_error().decode() or "distinct" in S._lib.sgm_last_error().decode()
    # a non-solenoidal source is refused by the check (SGM_E_SOURCE_DIVERGENCE = 6)
    assert pl.check_source(dev(np.random.default_rng(5).standard_normal(pl.N_e))) == 6


@pytest.mark.parametrize("p,n", [(2, (4, 3, 5)), (3, 5)])
def test_quadrature_rule_p_plus_2(p, n):
    """quad_points = p + 2 (sgm_plan_desc.quad_points; the generic CTA-per-element Hodge kernel) on the
    curved C3 map with a variable eps: Hodge stars and 20 steps against tier B built with the same
    (p + 2)-point rule (reading Z13: plan and oracle use the same rule)."""
    Q = p + 2
    ctrl = W.interpolate_map(p, n, W.c3_map)
    pl = S.Plan(n, p, geom_ctrl=ctrl, quad_points=Q)
    X = pl.qp_coords()
    eps = 1.0 + 0.5 * np.sin(2 * np.pi * X[:, 0]) * np.cos(2 * np.pi * X[:, 1])
    pl.set_material(S.EPS, eps)
    tb = TierB(p, n, ctrl=ctrl, inv_eps=1.0 / eps, inv_mu=1.0, Q=Q)
    g = np.random.default_rng(81)
    x = g.standard_normal(tb.N_e)
    y = torch.empty(tb.N_e, dtype=torch.float64, device="cuda")
    pl.hodge_star(S.MASS_EPS, dev(x), y)
    assert rel(host(y), tb.hodge_eps(x)) < 1e-11
    xb = g.standard_normal(tb.N_h)
    yb = torch.empty(tb.N_h, dtype=torch.float64, device="cuda")
    pl.hodge_star(S.MASS_MU, dev(xb), yb)
    assert rel(host(yb), tb.hodge_mu(xb)) < 1e-11
    st = _state(tb, 82)
    dt = 0.3 * W.cfl_dt_max(tb)
    for a, b in zip(_run_gpu(pl, st, dt, 20), tb.run(*st, dt, 20)):
        assert rel(a, b) < 1e-10


def test_c3_recipe_small():
    """The configs[2] recipe (oracle.workloads.c3_setup / c3_source: curved map, eps inclusion, projected
    Gaussian source, zero fields, Gaussian pulse in time) at 8^3, 60 steps through the pulse."""
    p, n = 3, 8
    ctrl, eps, _ = W.c3_setup(p, n)
    jhat = W.c3_source(p, n, ctrl)
    pl = S.Plan(n, p, geom_ctrl=ctrl)
    pl.set_material(S.EPS, eps)
    tb = TierB(p, n, ctrl=ctrl, inv_eps=1.0 / eps, inv_mu=1.0)
    dt = 0.5 * W.cfl_dt_max(tb)
    steps = 60
    jamp = W.c3_amplitudes(dt * 6, steps)  # the pulse (t0 = 0.15) inside the run
    st = tuple(np.zeros(k) for k in (tb.N_e, tb.N_e, tb.N_h, tb.N_h))
    out = _run_gpu(pl, st, dt, steps, jhat, jamp)
    for a, b in zip(out, tb.run(*st, dt, steps, jhat, jamp)):
        assert np.linalg.norm(b) > 0 and rel(a, b) < 1e-10


def test_pcg_star_zero_rhs_is_zero():
    """Scheme-1 PCG stars (curved map) on a zero right-hand side give exactly zero (a zero denominator
    in the CG ratios is a zero step, not NaN: ADVICE r1), and a zero-field start stays zero."""
    p, n = 3, 5
    pl = S.Plan(n, p, geom_ctrl=W.interpolate_map(p, n, W.c3_map))
    pl.set_scheme(1)
    z = torch.zeros(pl.N_e, dtype=torch.float64, device="cuda")
    y = torch.full((pl.N_e,), 7.0, dtype=torch.float64, device="cuda")
    pl.hodge_star(S.MASS_EPS, z, y)
    assert torch.count_nonzero(y).item() == 0
    st = [torch.zeros(k, dtype=torch.float64, device="cuda") for k in (pl.N_e, pl.N_e, pl.N_h, pl.N_h)]
    pl.step(*st, 0.001, 3)
    assert all(torch.isfinite(x).all().item() and torch.count_nonzero(x).item() == 0 for x in st)


@pytest.mark.parametrize("opts", [0, S.OPT_FUSED, S.OPT_FULL_SCHEDULE, S.OPT_FUSED | S.OPT_FULL_SCHEDULE])
@pytest.mark.parametrize("p,n", [(2, (5, 9, 7)), (3, 11), (4, (6, 5, 8))])
def test_eh_state_step(p, n, opts):
    """sgm_step_eh (the (e,h)-state variant, two stored vectors) against the oracle's step_eh with a
    divergence-free source and per-step amplitudes: 1 step <= 1e-11, 40 steps <= 1e-10."""
    pl = S.Plan(n, p)
    pl.set_options(opts)
    tb = TierB(p, n)
    g = np.random.default_rng(93)
    e0 = tb.hodge_eps(g.standard_normal(tb.N_e))
    h0 = tb.hodge_mu(g.standard_normal(tb.N_h))
    j = forms.join(curl_dual(tb.split_h(g.standard_normal(tb.N_h))))
    amp = np.cos(0.3 * np.arange(40))
    dt = 0.4 * W.cfl_dt_max(tb)
    for k, tol in ((1, 1e-11), (40, 1e-10)):
        e, h = dev(e0), dev(h0)
        pl.step_eh(e, h, dt, k, j_hat=dev(j), j_amp=dev(amp[:k]))
        er, hr = tb.run_eh(e0, h0, dt, k, j, amp[:k])
        assert rel(host(e), er) < tol and rel(host(h), hr) < tol, (k, rel(host(e), er), rel(host(h), hr))


def test_eh_state_general_hodge():
    """sgm_step_eh with a curved map and variable eps (general Hodge path, increments accumulated by
    the last solve sweep) against the oracle."""
    p, n = 3, 6
    ctrl = W.interpolate_map(p, n, W.c3_map)
    pl = S.Plan(n, p, geom_ctrl=ctrl)
    X = pl.qp_coords()
    eps = 1.0 + 0.5 * np.sin(2 * np.pi * X[:, 0])
    pl.set_material(S.EPS, eps)
    tb = TierB(p, n, ctrl=ctrl, inv_eps=1.0 / eps, inv_mu=1.0)
    g = np.random.default_rng(94)
    e0, h0 = tb.hodge_eps(g.standard_normal(tb.N_e)), tb.hodge_mu(g.standard_normal(tb.N_h))
    dt = 0.4 * W.cfl_dt_max(tb)
    e, h = dev(e0), dev(h0)
    pl.step_eh(e, h, dt, 20)
    er, hr = tb.run_eh(e0, h0, dt, 20)
    assert rel(host(e), er) < 1e-10 and rel(host(h), hr) < 1e-10


@pytest.mark.parametrize("n", [(3, 4, 2), (5, 6, 4)])
def test_lifted_coax_tem_step(n):
    """sgm_step_lifted on the coax (rational quarter annulus 1 < r < sqrt2; general Hodge with the
    full metric) with the TEM mode's inhomogeneous Dirichlet data on the symmetry planes (lifting,
    P:L450-490): 60 steps against the literal lifted tier A (full X^2_h, rectangular D1 / M2,
    (K1)_0 e_0 = M~2 d - (K1)_b e_b); the time-separable vectors are the caller's one-time setup."""
    from oracle import lifting as Lf
    p, dt, K = 2, 2e-3, 60
    A, st, g = Lf.coax_setup(p, n, dt)
    V = Lf.lifting_vectors(A, st[2], dt)
    gk = np.array([g((k + 1) * dt) for k in range(K)])
    beta = -dt * np.cumsum(gk)
    gg = A.ctrl
    pl = S.Plan(n, p, geom_ctrl=gg.P, geom_weights=gg.w)
    d, e, b, h = dev(st[0]), dev(st[1]), dev(st[2][A.b_int]), dev(st[3])
    pl.step_lifted(d, e, b, h, dt, K, dev(gk), dev(beta), w_e=dev(V["w_e"]), c_b=dev(V["c_b"]),
                   q0=dev(V["q0"]), q1=dev(V["q1"]))
    ref = A.run(*st, dt, K, g)
    for x, r in zip((d, e, b, h), (ref[0], ref[1], ref[2][A.b_int], ref[3])):
        assert rel(host(x), r) < 1e-10


def test_lifted_step_separable_cube():
    """sgm_step_lifted on the identity cube (separable reduced stars: the affine terms ride on the
    pipelined sweeps' stores) with synthetic lifting vectors, against the same recurrence in tier B."""
    p, n, K, dt = 3, (7, 6, 5), 25, 0.01
    pl = S.Plan(n, p)
    tb = TierB(p, n)
    g = np.random.default_rng(95)
    st = _state(tb, 96)
    st = (st[0], tb.hodge_eps(st[0]), st[2], tb.hodge_mu(st[2]))
    w_e, c_b = g.standard_normal(tb.N_e), g.standard_normal(tb.N_h)
    q0, q1 = g.standard_normal(tb.N_h), g.standard_normal(tb.N_h)
    gk = np.cos(0.2 * np.arange(1, K + 1))
    beta = -dt * np.cumsum(gk)
    dv = [dev(x) for x in st]
    pl.step_lifted(*dv, dt, K, dev(gk), dev(beta), w_e=dev(w_e), c_b=dev(c_b), q0=dev(q0), q1=dev(q1))
    d, e, b, h = st
    for k in range(K):
        d = d + dt * forms.join(curl_dual(tb.split_h(h)))
        e = tb.hodge_eps(d) - gk[k] * w_e
        b = b - dt * (forms.join(curl_primal(tb.split_e(e))) + gk[k] * c_b)
        h = tb.hodge_mu(b) + q0 + beta[k] * q1
    for x, r in zip(dv, (d, e, b, h)):
        assert rel(host(x), r) < 1e-10


@pytest.mark.parametrize("p,n", [(3, (17, 13, 23)), (4, (9, 10, 11)), (2, (21, 6, 30))])
def test_general_hodge_bitwise_reproducible(p, n):
    """The general (sum-factorised) Hodge accumulates element contributions through per-item output
    patches summed in a fixed order (no fp64 atomics): repeated applies, stars and steps are bitwise
    identical, and equal the oracle's mass apply (atomics made C3/C4 non-reproducible)."""
    ctrl = W.interpolate_map(p, n, W.c3_map)
    pl = S.Plan(n, p, geom_ctrl=ctrl)
    X = pl.qp_coords()
    eps = 1.0 + 0.5 * np.sin(2 * np.pi * X[:, 0]) * np.cos(2 * np.pi * X[:, 1])
    pl.set_material(S.EPS, eps)
    tb = TierB(p, n, ctrl=ctrl, inv_eps=1.0 / eps, inv_mu=1.0)
    g = np.random.default_rng(97)
    x = dev(g.standard_normal(tb.N_e))
    ys = []
    for _ in range(3):
        y = torch.empty_like(x)
        pl.hodge_apply(S.MASS_EPS, x, y)
        ys.append(y)
    assert all(torch.equal(ys[0], y) for y in ys[1:])
    assert rel(host(ys[0]), forms.join(tb.mass_eps(tb.split_e(host(x))))) < 1e-13
    st = _state(tb, 98)
    outs = []
    for _ in range(2):
        d, e, b, h = (dev(v) for v in st)
        pl.step(d, e, b, h, 0.001, 5)
        outs.append((d, e, b, h))
    assert all(torch.equal(a, b) for a, b in zip(*outs))


@pytest.mark.parametrize("p", [2, 3, 4])
@pytest.mark.parametrize("axis", [0, 1, 2])
def test_maximum_line_length(p, axis):
    """Lines of the maximum length the plan accepts (n_el + p - 1 = 392, include/sgm.h) along each
    axis: the sweeps fall back to a single slab and, where two line-operator tables do not fit
    together, to one launch per table (sweep_launch.cuh).  Hodge star and 3 steps against the oracle;
    scheme 1 at p = 4 (the p + 1 wide-band layout) as well."""
    from oracle.structured import TierB1
    n = [3, 2, 4]
    n[axis] = 393 - p
    n = tuple(n)
    schemes = (2, 1) if p == 4 else (2,)
    for scheme in schemes:
        pl = S.Plan(n, p)
        if scheme == 1:
            pl.set_scheme(1)
        tb = TierB(p, n) if scheme == 2 else TierB1(p, n)
        st = _state(tb, 31 + axis)
        y = torch.empty(tb.N_e, dtype=torch.float64, device="cuda")
        pl.hodge_star(S.MASS_EPS, dev(st[0]), y)
        assert rel(host(y), tb.hodge_eps(st[0])) < 1e-10, scheme
        dt = 0.05 / max(n)
        out = _run_gpu(pl, st, dt, 3)
        for a_, b_ in zip(out, tb.run(*st, dt, 3)):
            assert rel(a_, b_) < 1e-10, scheme


@pytest.mark.parametrize("p", [2, 3, 4])
@pytest.mark.parametrize("axis", [0, 1, 2])
def test_long_lines_windowed(p, axis):
    """Lines longer than one CTA holds (n_el + p - 1 > 392) are swept in overlapping windows of at
    most 14 segments (kernels.cu launch_sweep_windows): n_el = 512 along one axis (and 1000 along x at
    p = 3), every axis, p = 2-4.  Kronecker solves and transposes, Hodge stars, 3 steps and the full
    three-axis schedule against the oracle; scheme 1 at p = 3."""
    from oracle.structured import TierB1
    n = [3, 2, 4]
    n[axis] = 1000 if (p == 3 and axis == 0) else 512
    n = tuple(n)
    pl = S.Plan(n, p)
    tb = TierB(p, n)
    st = _state(tb, 61 + axis)
    g = np.random.default_rng(71 + axis)
    for which, N, split, solve in ((S.K1, tb.N_e, tb.split_e, tb.solve_K1), (S.KT1, tb.N_h, tb.split_h, tb.solve_Kt1)):
        for T in (False, True):
            r = g.standard_normal(N)
            x = torch.empty(N, dtype=torch.float64, device="cuda")
            pl.kron_solve(which, dev(r), x, transpose=T)
            assert rel(host(x), forms.join(solve(split(r), T=T))) < solve_tol(tb), (which, T)
    y = torch.empty(tb.N_e, dtype=torch.float64, device="cuda")
    pl.hodge_star(S.MASS_EPS, dev(st[0]), y)
    assert rel(host(y), tb.hodge_eps(st[0])) < 1e-10
    yh = torch.empty(tb.N_h, dtype=torch.float64, device="cuda")
    pl.hodge_star(S.MASS_MU, dev(st[2]), yh)
    assert rel(host(yh), tb.hodge_mu(st[2])) < 1e-10
    dt = 0.05 / max(n)
    ref = tb.run(*st, dt, 3)
    for opts in (0, S.OPT_FULL_SCHEDULE):
        pl.set_options(opts)
        out = _run_gpu(pl, st, dt, 3)
        for a_, b_ in zip(out, ref):
            assert rel(a_, b_) < 1e-10, opts
    pl.set_options(0)
    if p == 3:
        pl1 = S.Plan(n, p)
        pl1.set_scheme(1)
        tb1 = TierB1(p, n)
        out = _run_gpu(pl1, st, dt, 3)
        for a_, b_ in zip(out, tb1.run(*st, dt, 3)):
            assert rel(a_, b_) < 1e-10


@pytest.mark.parametrize("p,n", [(2, (6, 5, 7)), (3, (9, 10, 11)), (3, (6, 5, 7)), (4, (5, 6, 4))])
def test_otf_geometry_parity(p, n):
    """On-the-fly DF in the general Hodge (SGM_OPT_OTF_GEOMETRY): the brick kernel
    evaluates DF at the quadrature points from the map's control points and forms the 2-form
    weights itself (1 stored double per point instead of 6).  Curved polynomial map, variable eps,
    ragged bricks: both Hodge applies against the oracle and against the stored-W kernel, 1 and 20
    steps against the oracle, bitwise-repeatable applies; clearing the option restores stored W."""
    ctrl, eps = _curved_case(p, n)
    tb = TierB(p, n, ctrl=ctrl, inv_eps=1.0 / eps, inv_mu=1.0)
    tb.sep_mu = None
    tb.W_mu = tb._W(1.0)
    ref = S.Plan(n, p, geom_ctrl=ctrl)
    ref.set_material(S.EPS, eps)
    pl = S.Plan(n, p, geom_ctrl=ctrl)
    pl.set_material(S.EPS, eps)
    pl.set_options(S.OPT_OTF_GEOMETRY)  # rebuilds both general stars from the stored material
    assert pl.options() == S.OPT_OTF_GEOMETRY
    g = np.random.default_rng(131)
    for which, N, mass, split in ((S.MASS_EPS, tb.N_e, tb.mass_eps, tb.split_e),
                                  (S.MASS_MU, tb.N_h, tb.mass_mu, tb.split_h)):
        x = g.standard_normal(N)
        ys = []
        for plan in (pl, pl, ref):
            y = torch.empty(N, dtype=torch.float64, device="cuda")
            plan.hodge_apply(which, dev(x), y)
            ys.append(y)
        assert torch.equal(ys[0], ys[1])
        assert rel(host(ys[0]), forms.join(mass(split(x)))) < 1e-13
        assert rel(host(ys[0]), host(ys[2])) < 1e-14
    st = _state(tb, 132)
    dt = 0.02 / max(forms._n3(n))
    for k, tol in ((1, 1e-11), (20, 1e-10)):
        out = _run_gpu(pl, st, dt, k)
        for a, b in zip(out, tb.run(*st, dt, k)):
            assert rel(a, b) < tol
    # the option set before the material: the material upload builds the on-the-fly form directly
    pl2 = S.Plan(n, p, geom_ctrl=ctrl)
    pl2.set_options(S.OPT_OTF_GEOMETRY)
    pl2.set_material(S.EPS, eps)
    x = g.standard_normal(tb.N_e)
    y2 = torch.empty(tb.N_e, dtype=torch.float64, device="cuda")
    pl2.hodge_apply(S.MASS_EPS, dev(x), y2)
    y1 = torch.empty_like(y2)
    pl.hodge_apply(S.MASS_EPS, dev(x), y1)
    assert torch.equal(y1, y2)
    # cleared: the stored 6-entry weights again, bitwise equal to a plan that never had the option
    pl.set_options(0)
    y0 = torch.empty_like(y2)
    ref.hodge_apply(S.MASS_EPS, dev(x), y0)
    pl.hodge_apply(S.MASS_EPS, dev(x), y1)
    assert torch.equal(y0, y1)
