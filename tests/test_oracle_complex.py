"""Pins of the oracle's 3D layer: incidence matrices, pairings and 2-form masses (tier A).

Paper facts used: d o d = 0; dim X^k_{h,0} = dim X~^{3-k};
K~_{3-k} = K_k^T; discrete integration by parts; Kronecker block
structure; metric independence of pairings.  Mass facts are
mathematics: SPD, Kronecker product of 1D Grams for constant material on the identity map,
exact scaling under a diagonal affine map, linearity in the material.
"""
import numpy as np
import pytest
import scipy.sparse as sp

from oracle import forms
from oracle import workloads as W
from oracle.assemble import Quad, pairing, mass2, identity_ctrl, physical_qp
from oracle.splines import gram_1d


CASES = [(2, 2), (3, 3), (4, 2), (2, (2, 3, 4))]


def test_dimension_examples():
    # S:L129 example: p=2, n=2 -> dim X^1_{h,0} = 36 = dim X~^2
    assert forms.form_dim("primal", 1, 2, 2) == 36
    assert forms.form_dim("dual", 2, 2, 2) == 36
    # C_1 is 12 x 12 at p=2, n=2
    assert np.prod(forms.component_shapes("primal", 1, 2, 2)[0]) == 12


@pytest.mark.parametrize("p,n", CASES)
def test_dimension_duality(p, n):
    for k in range(4):
        assert forms.form_dim("primal", k, p, n) == forms.form_dim("dual", 3 - k, p, n)


@pytest.mark.parametrize("p,n", CASES)
def test_d_d_zero_exact_integers(p, n):
    for cplx in ("primal", "dual"):
        for k in range(2):
            A = forms.incidence(cplx, k, p, n)
            B = forms.incidence(cplx, k + 1, p, n)
            assert A.dtype == np.int64 and B.dtype == np.int64
            assert abs(B @ A).max() == 0
            assert set(np.unique(A.data)) <= {-1, 1}


@pytest.mark.parametrize("p,n", CASES)
def test_dual_curl_is_transpose_of_primal_curl(p, n):
    """D~1 = (D1)^T exactly; gradient/divergence pair up with a minus sign."""
    D0, D1, D2 = (forms.incidence("primal", k, p, n) for k in range(3))
    Dt0, Dt1, Dt2 = (forms.incidence("dual", k, p, n) for k in range(3))
    assert abs(Dt1 - D1.T).max() == 0
    assert abs(Dt2 + D0.T).max() == 0
    assert abs(Dt0 + D2.T).max() == 0


def test_univariate_factor_example():
    # S:L18 example: rows [-1 1 0 0; 0 -1 1 0; 0 0 -1 1] for S_p -> S_{p-1} untrimmed, m = 4.
    # Our trimmed primal factor is the same stencil restricted to interior columns; the dual
    # factor (dv)_j = v_{j+1} - v_j is exactly that matrix.
    Dt = forms.incidence("dual", 0, 3, (2, 1, 1))   # b = 4 along x, a = 3 -> x-component rows
    Dx = Dt[:3, :].toarray()
    # first component of the dual gradient acting on x only for the first (y,z) line
    assert np.array_equal(Dx[:, :4], np.array([[-1, 1, 0, 0], [0, -1, 1, 0], [0, 0, -1, 1]]))


@pytest.mark.parametrize("p,n", CASES)
def test_pairing_transpose_and_integration_by_parts(p, n):
    q = Quad(p, n)
    K = {k: pairing(q, f"K{k}") for k in range(4)}
    Kt = {k: pairing(q, f"Kt{k}") for k in range(4)}
    for k in range(4):
        # eq. pairing_transpose: K~_{3-k} = K_k^T
        assert abs(Kt[3 - k] - K[k].T).max() < 1e-15
    D = {k: forms.incidence("primal", k, p, n) for k in range(3)}
    Dt = {k: forms.incidence("dual", k, p, n) for k in range(3)}
    for k in (1, 2, 3):
        # eq. disc_int_by_parts2: (D~^{3-k})^T K_{k-1} = (-1)^{3-k+1} K_k D^{k-1}
        lhs = Dt[3 - k].T @ K[k - 1]
        rhs = (-1) ** (3 - k + 1) * (K[k] @ D[k - 1])
        assert abs(lhs - rhs).max() < 1e-14
        # eq. disc_int_by_parts1: (D^{k-1})^T K~_{3-k} = (-1)^k K~_{3-k+1} D~^{3-k}
        lhs = D[k - 1].T @ Kt[3 - k]
        rhs = (-1) ** k * (Kt[3 - k + 1] @ Dt[3 - k])
        assert abs(lhs - rhs).max() < 1e-14


@pytest.mark.parametrize("p,n", CASES)
def test_pairing_blocks_are_kronecker_products(p, n):
    """3D-quadrature K1 blocks = G^3 (x) G^2 (x) M^1 etc. (eq. tensor_K / tensor_Ktilde)."""
    q = Quad(p, n)
    n3 = forms._n3(n)
    G = [gram_1d("Dp2", "Sp", p, n3[a]) for a in range(3)]
    M = [gram_1d("Dp1", "Sp1", p, n3[a]) for a in range(3)]
    K1 = pairing(q, "K1")
    Kt1 = pairing(q, "Kt1")
    oe = forms.offsets("primal", 1, p, n3)
    oh = forms.offsets("dual", 1, p, n3)
    for c in range(3):
        A = [M[a] if a == c else G[a] for a in range(3)]
        C = np.kron(A[2], np.kron(A[1], A[0]))
        assert np.abs(K1[oe[c]:oe[c + 1], oe[c]:oe[c + 1]].toarray() - C).max() < 1e-15
        B = [G[a].T if a == c else M[a].T for a in range(3)]
        Ct = np.kron(B[2], np.kron(B[1], B[0]))
        assert np.abs(Kt1[oh[c]:oh[c + 1], oh[c]:oh[c + 1]].toarray() - Ct).max() < 1e-15


def _c3_ctrl(p, n):
    return W.interpolate_map(p, n, W.c3_map)


@pytest.mark.parametrize("p,n", [(2, 2), (3, 2)])
def test_pairing_metric_independence(p, n):
    """Assembling K1 / K~1 with physical pull-backs on the C3 map gives the parametric matrices
    (S:L247)."""
    q = Quad(p, n)
    ctrl = _c3_ctrl(p, n)
    for which in ("K1", "Kt1"):
        A = pairing(q, which)
        B = pairing(q, which, ctrl=ctrl, physical=True)
        assert abs(A - B).max() < 1e-14


@pytest.mark.parametrize("p,n", [(2, 2), (3, 2), (4, 1)])
def test_mass_identity_kronecker_and_affine(p, n):
    q = Quad(p, n)
    gam = 0.37
    Md = mass2(q, "dual", np.full(q.nqp, gam))
    Mp = mass2(q, "primal", np.full(q.nqp, gam))
    oe = forms.offsets("dual", 2, p, n)
    ob = forms.offsets("primal", 2, p, n)
    GB1, GC2 = gram_1d("Dp1", "Dp1", p, n), gram_1d("Dp2", "Dp2", p, n)
    GBp, GC1 = gram_1d("Sp", "Sp", p, n), gram_1d("Sp1", "Sp1", p, n)
    for c in range(3):
        A = [GB1 if a == c else GC2 for a in range(3)]
        assert np.abs(Md[oe[c]:oe[c + 1], oe[c]:oe[c + 1]].toarray()
                      - gam * np.kron(A[2], np.kron(A[1], A[0]))).max() < 1e-15
        B = [GBp if a == c else GC1 for a in range(3)]
        assert np.abs(Mp[ob[c]:ob[c + 1], ob[c]:ob[c + 1]].toarray()
                      - gam * np.kron(B[2], np.kron(B[1], B[0]))).max() < 1e-15
    # off-diagonal component blocks vanish for the identity map
    assert abs(Md[oe[0]:oe[1], oe[1]:oe[2]]).max() < 1e-16
    # diagonal affine map F = diag(L) x: block c scales by L_c^2 / (Lx Ly Lz)
    L = np.array([2.0, 0.5, 1.5])
    ctrl = identity_ctrl(p, n) * L
    Ma = mass2(q, "dual", None, ctrl)
    M1 = mass2(q, "dual", None, None)
    for c in range(3):
        s = L[c] ** 2 / np.prod(L)
        blk = slice(oe[c], oe[c + 1])
        assert np.abs(Ma[blk, blk] - s * M1[blk, blk]).max() < 1e-14
    # SPD and linearity in gamma
    g = np.random.default_rng(4).uniform(0.5, 2.0, q.nqp)
    Mg = mass2(q, "dual", g, _c3_ctrl(p, n))
    assert abs(Mg - Mg.T).max() < 1e-15
    assert np.linalg.eigvalsh(Mg.toarray()).min() > 0
    M2g = mass2(q, "dual", 2 * g + 0.5, _c3_ctrl(p, n))
    Mh = mass2(q, "dual", np.full(q.nqp, 0.5), _c3_ctrl(p, n))
    assert abs(M2g - (2 * Mg + Mh)).max() < 1e-14


def test_physical_points_agree():
    p, n = 3, 2
    ctrl = _c3_ctrl(p, n)
    q = Quad(p, n)
    A = physical_qp(q, ctrl).reshape(-1, 3)
    B = W.physical_points(p, n, ctrl)
    Bel = np.stack([W.grid_to_elem(B[..., i], n, p + 1) for i in range(3)], -1)
    assert np.abs(A - Bel).max() < 1e-14
    # the interpolated C3 map reproduces the analytic map at Greville points exactly and
    # keeps the boundary of the unit cube fixed: corner control points are the corners
    assert np.abs(ctrl[0, 0, 0]).max() < 1e-15 and np.abs(ctrl[-1, -1, -1] - 1).max() < 1e-14
