"""Oracle pins against the fixtures in tests/golden/ (each fixture cites its passage).

* cavity_spectrum.json: the discrete scheme-2 operator reproduces the exact PEC-cube spectrum
   with the right multiplicities, converges at the rate of the H-side spaces, and has the
  discrete gradients as its exact null space.
* bernstein_1d.json / dimensions.json: closed forms and worked examples of the 1D factors and the
  complexes.
"""
import json
import os

import numpy as np
import pytest

from oracle import forms
from oracle.splines import gram_1d, open_knots
from oracle.structured import TierB, curl_primal, curl_dual

G = os.path.join(os.path.dirname(__file__), "golden")


def load(name):
    return json.load(open(os.path.join(G, name)))


def leapfrog_operator(p, n):
    """Dense A = D~1 K~1^{-1} M2 D1 K1^{-1} M~2 on X~2 (the d-form of scheme 2)."""
    tb = TierB(p, n)
    N = tb.N_e
    A = np.zeros((N, N))
    I = np.eye(N)
    for i in range(N):
        e = tb.solve_K1(tb.mass_eps(tb.split_e(I[:, i])))
        h = tb.solve_Kt1(tb.mass_mu(curl_primal(e)))
        A[:, i] = forms.join(curl_dual(h))
    return A


@pytest.mark.parametrize("p,n,tol", [(2, 4, 0.12), (3, 4, 2e-3), (4, 3, 1e-3)])
def test_cavity_spectrum(p, n, tol):
    gold = load("cavity_spectrum.json")
    ev = np.linalg.eigvals(leapfrog_operator(p, n))
    assert np.max(np.abs(ev.imag)) < 1e-9 * np.max(np.abs(ev))
    ev = np.sort(ev.real)
    a = n + p - 2
    scale = np.max(ev)
    zeros = np.sum(np.abs(ev) < 1e-10 * scale)
    assert zeros == eval(gold["null_space_dim_formula"], {"n": n, "p": p})  # = dim im D0 = a^3
    nz = ev[ev > 1e-10 * scale]
    ref = np.array(gold["eigenvalues_over_pi2"], dtype=float) * np.pi ** 2
    got = nz[:len(ref)]
    # the two lowest families (2 pi^2, three-fold; 3 pi^2, two-fold) to the mesh accuracy
    assert np.all(np.abs(got[:5] - ref[:5]) / ref[:5] < tol), (got / np.pi ** 2)
    # approximation from above, and the exact multiplicities of the first three families
    assert np.all(got[:5] >= ref[:5] * (1 - 1e-12))
    for lo, hi in ((0, 3), (3, 5), (5, 11)):
        cl = got[lo:hi]
        assert np.ptp(cl) < 1e-9 * cl[0], (lo, hi, cl)
    assert got[5] > got[4] * (1 + 1e-6) and got[11] > got[10] * (1 + 1e-6)
    assert a ** 3 == zeros


def test_cavity_spectrum_convergence_rate():
    """Eigenvalue error of the first mode ~ h^(2(p-1)) (the H-side spaces have degree p-1)."""
    gold = load("cavity_spectrum.json")
    lam = gold["eigenvalues_over_pi2"][0] * np.pi ** 2
    errs = []
    for n in (3, 4):
        ev = np.sort(np.linalg.eigvals(leapfrog_operator(3, n)).real)
        nz = ev[ev > 1e-10 * ev[-1]]
        errs.append(nz[0] - lam)
    rate = np.log(errs[0] / errs[1]) / np.log(4 / 3)
    assert 3.3 < rate < 5.0, rate


def test_bernstein_1d():
    gold = load("bernstein_1d.json")
    assert np.allclose(gram_1d("Dp2", "Sp", 2, 1), gold["p2"]["G"], rtol=0, atol=1e-15)
    assert np.allclose(gram_1d("Dp1", "Sp1", 2, 1), gold["p2"]["M"], rtol=0, atol=1e-15)
    assert abs(gram_1d("Sp", "Sp", 2, 1)[0, 0] - gold["p2_gamma_Bp_n1"]) < 1e-15


def test_dimensions():
    gold = load("dimensions.json")
    for k in gold["knots"]:
        kv = open_knots(k["p"], k["n"])
        if "knots" in k:
            assert np.allclose(kv, k["knots"])
        assert len(kv) - k["p"] - 1 == k["dim"]
    for f in gold["forms"]:
        assert forms.form_dim(f["cplx"], f["k"], f["p"], f["n"]) == f["dim"], f
    c = gold["K1_block_C1"]
    assert int(np.prod(forms.component_shapes("primal", 1, c["p"], c["n"])[0])) == c["size"]


def test_curved_map_converges_to_cube_spectrum():
    """SURVEY 8(c) physics pin: the C3 map sends the unit cube onto itself, so with eps = mu = 1 the
    discrete spectrum on the curved mesh converges to the same exact cavity spectrum:
    the five lowest eigenvalues -> (2, 2, 2, 3, 3) pi^2 with error ~ h^(2(p-1)) (the map breaks the
    cube's symmetry, so the multiplicities split at finite h)."""
    from oracle import workloads as W
    gold = load("cavity_spectrum.json")
    ref = np.array(gold["eigenvalues_over_pi2"][:5], dtype=float) * np.pi ** 2
    p, errs = 3, []
    for n in (3, 4, 5):
        tb = TierB(p, n, ctrl=W.interpolate_map(p, n, W.c3_map))
        N = tb.N_e
        A = np.zeros((N, N))
        I = np.eye(N)
        for i in range(N):
            e = tb.solve_K1(tb.mass_eps(tb.split_e(I[:, i])))
            h = tb.solve_Kt1(tb.mass_mu(curl_primal(e)))
            A[:, i] = forms.join(curl_dual(h))
        ev = np.sort(np.linalg.eigvals(A).real)
        got = ev[ev > 1e-10 * ev[-1]][:5]
        assert np.all(got >= ref * (1 - 1e-12))
        errs.append(np.max(np.abs(got - ref) / ref))
    rates = [np.log(errs[0] / errs[1]) / np.log(4 / 3), np.log(errs[1] / errs[2]) / np.log(5 / 4)]
    assert errs[-1] < 2e-3 and all(3.3 < r < 5.0 for r in rates), (errs, rates)


def test_c3_source_fixture_is_the_oracle_recipe():
    """tests/golden/c3_a_hat.npz (read by bench.py for the C3 source) is exactly what
    scripts/make_c3_source.py computes from the oracle (readings Z16/Z28), and its dual curl is the
    divergence-free j^ of oracle.workloads.c3_source."""
    import synth
    from oracle import workloads as W
    from oracle.structured import curl_dual, div_dual
    z = np.load(os.path.join(G, "c3_a_hat.npz"))
    p, n = int(z["p"]), int(z["n"])
    ctrl, _, _ = W.c3_setup(p, n)
    _, c_J = synth.c3_centres()
    a = W.project_dual1(p, n, synth.gaussian_z(W.physical_points(p, n, ctrl), c_J, W.C3_SIGMA))
    assert np.array_equal(a, z["a_hat"])
    j = forms.join(curl_dual(forms.split(a, "dual", 1, p, (n, n, n))))
    assert np.array_equal(j, W.c3_source(p, n, ctrl))
    assert np.abs(div_dual(forms.split(j, "primal", 1, p, (n, n, n)))).max() <= 1e-12 * np.abs(j).max()


def test_workload_dt_fixture():
    """tests/golden/workload_dt.json (scripts/make_workload_dt.py, oracle power iteration) holds
    dt = dt_max / 2 for each config, C1's dt_max agrees with SURVEY 8(d)'s derived 0.03807, and the
    quotient has converged to 1e-4 (monotone power iteration, reading Z15)."""
    d = load("workload_dt.json")
    assert abs(d["c1"]["dt_max"] - 0.03807) < 1e-4
    for k, v in d.items():
        if k.startswith("_"):
            continue
        assert abs(v["dt"] - 0.5 * v["dt_max"]) < 1e-15 * v["dt"]
        assert abs(v["dt_max"] - 2.0 / np.sqrt(v["lambda"])) < 1e-12 * v["dt_max"]
        assert -1e-12 * v["lambda"] <= v["lambda"] - v["lambda_prev"] < 1e-4 * v["lambda"]
