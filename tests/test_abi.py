"""CPU-side checks of the C ABI: the library loads, exports every symbol include/sgm.h declares,
and the host setup logic (1D tables, shapes, quadrature coordinates, classification, error
codes) agrees with the oracle.  No kernel is launched here."""
import ctypes
import os
import re
import sys

import numpy as np
import pytest

import paper_2302_04979_b200 as S
from oracle import forms
from oracle import workloads as W
from oracle.splines import gram_1d

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    txt = open(os.path.join(ROOT, "include", "sgm.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(sgm_[a-z_0-9]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    names = _declared()
    assert len(names) >= 20
    lib = ctypes.CDLL(S.LIB_PATH)
    for nm in names:
        assert hasattr(lib, nm), nm
        assert nm in S.EXPORTED, nm
    assert S.sgm_version().decode().startswith("sgm")


@pytest.mark.parametrize("p,n", [(2, 4), (3, (5, 3, 4)), (4, 7)])
def test_host_tables_match_oracle(p, n):
    pl = S.Plan(n, p, device=-1)
    n3 = forms._n3(n)
    spaces = [("Dp2", "Sp"), ("Dp1", "Sp1"), ("Dp1", "Dp1"), ("Dp2", "Dp2"), ("Sp", "Sp"), ("Sp1", "Sp1")]
    for ax in range(3):
        for which, (r, c) in enumerate(spaces):
            B = gram_1d(r, c, p, n3[ax])
            assert np.abs(pl.table(which, ax) - B).max() < 1e-14 * max(1.0, np.abs(B).max())


@pytest.mark.parametrize("p,n", [(2, 4), (3, (5, 3, 4))])
def test_shapes_and_lengths(p, n):
    pl = S.Plan(n, p, device=-1)
    assert pl.N_e == forms.form_dim("primal", 1, p, n) == forms.form_dim("dual", 2, p, n)
    assert pl.N_h == forms.form_dim("dual", 1, p, n) == forms.form_dim("primal", 2, p, n)
    for c in range(3):
        assert pl.shape(S.FORM_E, c) == forms.component_shapes("primal", 1, p, n)[c]
        assert pl.shape(S.FORM_D, c) == forms.component_shapes("dual", 2, p, n)[c]
        assert pl.shape(S.FORM_B, c) == forms.component_shapes("primal", 2, p, n)[c]
        assert pl.shape(S.FORM_H, c) == forms.component_shapes("dual", 1, p, n)[c]


def test_qp_coords_identity_and_curved():
    p, n = 3, (3, 2, 4)
    pl = S.Plan(n, p, device=-1)
    X = W.physical_points(p, n)
    Xel = np.stack([W.grid_to_elem(X[..., i], n, p + 1) for i in range(3)], -1)
    assert np.abs(pl.qp_coords() - Xel).max() < 1e-15
    ctrl = W.interpolate_map(p, n, W.c3_map)
    pl2 = S.Plan(n, p, geom_ctrl=ctrl, device=-1)
    X2 = W.physical_points(p, n, ctrl)
    X2el = np.stack([W.grid_to_elem(X2[..., i], n, p + 1) for i in range(3)], -1)
    assert np.abs(pl2.qp_coords() - X2el).max() < 1e-14
    assert not pl2.separable(S.MASS_EPS)
    assert pl.separable(S.MASS_EPS) and pl.separable(S.MASS_MU)


def test_classification_affine_and_material():
    from oracle.assemble import identity_ctrl
    p, n = 2, 3
    ctrl = identity_ctrl(p, n) * np.array([2.0, 0.5, 1.5])
    pl = S.Plan(n, p, geom_ctrl=ctrl, device=-1)
    assert pl.separable(S.MASS_EPS)        # axis-aligned affine + constant material
    pl.set_material(S.EPS, np.full(pl.qp_count(), 2.0))
    assert not pl.separable(S.MASS_EPS)    # variable material -> quadrature weights
    assert pl.separable(S.MASS_MU)


def test_error_codes():
    desc = S.sgm_plan_desc((ctypes.c_int * 3)(4, 4, 4), 1, None, 0, -1)
    h = ctypes.c_void_p()
    assert S.sgm_plan_create(ctypes.byref(desc), ctypes.byref(h)) == 2      # p < 2: unsupported
    desc = S.sgm_plan_desc((ctypes.c_int * 3)(0, 4, 4), 3, None, 0, -1)
    assert S.sgm_plan_create(ctypes.byref(desc), ctypes.byref(h)) == 1      # n_el < 1
    desc = S.sgm_plan_desc((ctypes.c_int * 3)(4, 4, 4), 3, None, 2, -1)
    assert S.sgm_plan_create(ctypes.byref(desc), ctypes.byref(h)) == 1      # Q < p+1
    # a form component above 2^31 - 2^20 elements (32-bit indices): unsupported
    desc = S.sgm_plan_desc((ctypes.c_int * 3)(1300, 1300, 1300), 3, None, 0, -1)
    assert S.sgm_plan_create(ctypes.byref(desc), ctypes.byref(h)) == 2
    # inverted geometry: det DF < 0
    from oracle.assemble import identity_ctrl
    ctrl = identity_ctrl(2, 3).copy()
    ctrl[..., 0] *= -1.0
    with pytest.raises(S.SgmError) as ei:
        S.Plan(3, 2, geom_ctrl=ctrl, device=-1)
    assert ei.value.status == 3
    pl = S.Plan(3, 2, device=-1)
    with pytest.raises(S.SgmError) as ei:
        pl.set_material(S.EPS, -np.ones(pl.qp_count()))
    # host-only plans classify but cannot validate device work; material validation happens
    # on device plans (build_mass); device calls on a host-only plan are rejected:
    rc = S.sgm_step(pl.h, 8, 16, 24, 32, None, None, 0.1, 1, 64, 1 << 20, None)
    assert rc == 1


def test_plain_c_consumer(tmp_path):
    """The library is a C ABI: a plain C program compiled against include/sgm.h links libsgm.so and
    runs host-side queries (no Python, no torch)."""
    import shutil
    import subprocess
    gcc = shutil.which("gcc")
    if gcc is None:
        pytest.skip("gcc not available")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    libdir = os.path.join(root, "paper_2302_04979_b200")
    exe = str(tmp_path / "abi_smoke")
    subprocess.run([gcc, "-std=c99", "-O1", os.path.join(root, "tests", "c", "abi_smoke.c"), "-I",
                    os.path.join(root, "include"), "-L", libdir, "-lsgm", "-Wl,-rpath," + libdir, "-o", exe],
                   check=True)
    r = subprocess.run([exe], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "abi_smoke ok" in r.stdout


@pytest.mark.parametrize("p,n", [(2, 5), (3, (9, 7, 6)), (4, 6), (3, 128)])
def test_reduced_schedule_identities_hold(p, n):
    """The plan verifies Hat M = Gamma_B^{p-1} diag(s) and Gamma_C^{p-1} = diag(s) Gamma_B^{p-1} diag(s)
    on every axis (host_setup.cpp) and enables the reduced separable schedule (fused direct sweeps by
    default); SGM_OPT_FULL_SCHEDULE selects the three-axis schedule, SGM_OPT_FUSED the fused update."""
    pl = S.Plan(n, p, device=-1)
    assert pl.reduced_schedule() and pl.schedule_mode() in (1, 2)
    pl.set_options(S.OPT_FULL_SCHEDULE)
    assert pl.options() == S.OPT_FULL_SCHEDULE and not pl.reduced_schedule()
    pl.set_options(S.OPT_FUSED)
    assert pl.schedule_mode() == 3
    pl.set_options(S.OPT_SERIAL)
    assert pl.schedule_mode() == 1
    pl.set_options(S.OPT_OTF_GEOMETRY)  # host-only plan: recorded, no weights to rebuild
    assert pl.options() == S.OPT_OTF_GEOMETRY and pl.reduced_schedule()
    with pytest.raises(S.SgmError):
        pl.set_options(0x100)


def test_kernels_per_step_fused_schedule():
    """The default step launches 7 kernels for separable stars on a cube (update, three eps sweep
    launches, update, two mu sweep launches); with the fused update (SGM_OPT_FUSED) 4 (the Ampere
    update fused into the first eps launch, the two concurrent second eps launches, the Faraday update
    fused into the mu launch); a fused launch carries at most two distinct line-operator tables, so
    three different element counts split the mu launch in two."""
    pl = S.Plan(32, 3, device=-1)
    assert pl.kernels_per_step() == 7
    pl.set_options(S.OPT_FUSED)
    assert pl.kernels_per_step() == 4
    pl.set_options(S.OPT_FUSED | S.OPT_FULL_SCHEDULE)
    assert pl.kernels_per_step() == 6
    for n, k in (((20, 21, 20), 4), ((20, 21, 22), 5)):
        pl = S.Plan(n, 3, device=-1)
        pl.set_options(S.OPT_FUSED)
        assert pl.kernels_per_step() == k


def test_product_library_ignores_tuning_environment():
    """The tuning knobs (SGM_PIPE_DBG, SGM_NODIAG, SGM_FORK, ... of the round-1 build) are compiled
    only into a -DSGM_TUNING build: the product library contains none of their names, so no
    environment variable can change its schedule or skip work; and a plan created with such
    variables set is the default plan."""
    import os
    import subprocess
    out = subprocess.run(["strings", S.LIB_PATH], capture_output=True, text=True, check=True).stdout
    knobs = sorted({w for w in out.splitlines() if re.fullmatch(r"SGM_[A-Z0-9_]+", w.strip())})
    assert knobs == [], knobs
    env = dict(os.environ, SGM_NODIAG="1", SGM_PIPE_DBG="15", SGM_FORK="0", SGM_SPIKE_FULL="1", SGM_SEG="28")
    code = ("import paper_2302_04979_b200 as S; pl = S.Plan(32, 3, device=-1); "
            "print(pl.schedule_mode(), pl.kernels_per_step(), pl.options())")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, cwd=ROOT)
    assert r.stdout.split() == ["2", "7", "0"], r.stdout + r.stderr


def test_verification_build_is_separate():
    """The protocol checks of csrc/check.cuh live only in libsgm_checked.so: the product library
    answers sgm_check_read with SGM_E_UNSUPPORTED (and reads no SGM_CHECK_INJECT, see above); the
    verification build, when present, exports the same C ABI."""
    n, f = ctypes.c_uint(7), ctypes.c_uint(7)
    assert S.sgm_check_read(1, ctypes.byref(n), ctypes.byref(f)) == 2
    assert (n.value, f.value) == (7, 7)
    assert "checked" not in S.sgm_version().decode()
    chk = os.path.join(os.path.dirname(S.LIB_PATH), "libsgm_checked.so")
    if os.path.exists(chk):
        lib = ctypes.CDLL(chk)
        for nm in _declared():
            assert hasattr(lib, nm), nm
        lib.sgm_version.restype = ctypes.c_char_p
        assert b"checked" in lib.sgm_version()


def test_rational_map_host_geometry():
    """A rational (NURBS) map through the C ABI: the plan's physical quadrature points equal the
    oracle's quotient-rule evaluation (quarter annulus), the Hodge stars are general, and
    non-positive weights are refused with SGM_E_GEOMETRY."""
    from oracle import workloads as W
    from oracle.assemble import Quad, physical_qp
    n = (2, 3, 2)
    g = W.quarter_annulus(n)
    pl = S.Plan(n, 2, geom_ctrl=g, device=-1)
    assert np.abs(pl.qp_coords() - physical_qp(Quad(2, n), g).reshape(-1, 3)).max() < 1e-15
    assert not pl.separable(S.MASS_EPS) and not pl.separable(S.MASS_MU)
    w = g.w.copy()
    w[0, 1, 1] = -1.0
    with pytest.raises(S.SgmError) as ei:
        S.Plan(n, 2, geom_ctrl=g.P, geom_weights=w, device=-1)
    assert "SGM_E_GEOMETRY" in str(ei.value)


def test_scheme_selection_rules():
    """sgm_plan_set_scheme: scheme 1 for every compiled degree (its eps star uses a p+1 table layout);
    curved maps and variable materials select the PCG stars; other values are refused."""
    S.Plan(6, 3, device=-1).set_scheme(1)
    S.Plan((3, 4, 5), 2, device=-1).set_scheme(1)
    S.Plan(3, 2, geom_ctrl=W_curved(2, 3), device=-1).set_scheme(1)
    S.Plan(6, 4, device=-1).set_scheme(1)
    pl = S.Plan(3, 2, device=-1)
    pl.set_scheme(1)
    pl.set_material(S.EPS, np.ones(pl.qp_count()))
    pl.set_scheme(2)
    with pytest.raises(S.SgmError):
        pl.set_scheme(3)


def W_curved(p, n):
    from oracle import workloads as W
    return W.interpolate_map(p, n, W.c3_map)


@pytest.mark.parametrize("p,n", [(2, 3), (3, (4, 5, 3)), (4, 6)])
def test_library_geometry_interpolation(p, n):
    """sgm_geometry_interpolate (used by bench.py for the C3 map) equals the oracle's Greville
    interpolation, and synth.c3_map equals the oracle's C3 map."""
    import synth
    from oracle import workloads as W
    a = S.interpolate_geometry(n, p, synth.c3_map)
    assert np.abs(a - W.interpolate_map(p, n, W.c3_map)).max() < 1e-13
    X = np.random.default_rng(3).uniform(size=(7, 3))
    assert np.array_equal(synth.c3_map(X), W.c3_map(X))


def test_long_lines_accepted():
    """Lines above 392 rows are swept in overlapping windows (launch_sweep): plans with n_el + p - 1
    above 392 along an axis are accepted (the round-1 limit), up to the 32-bit component limit."""
    for p, n in ((2, (1000, 3, 3)), (3, (3, 700, 4)), (4, (3, 3, 1200))):
        pl = S.Plan(n, p, device=-1)
        assert max(max(pl.shape(S.FORM_E, c)) for c in range(3)) == max(n) + p - 1
