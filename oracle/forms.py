"""Discrete form spaces and integer incidence matrices (TEST INFRASTRUCTURE ONLY).

PAPER.md sec. 2.3: primal complex X^k_{h,0} of mixed degree p / p-1 with the
first and last functions of S_p removed; dual complex X~^k of degree p-1 / p-2, free.
Component pattern of sec. 4.1: primal 1-form component c has the
degree-(p-1) space along axis c and the degree-p space along the other two axes; 2-forms
have the complementary pattern.

Vector layout: components 1,2,3 concatenated; each component a C-order
array [z][y][x] (x fastest), flat index  ix + nx*(iy + ny*iz).

The incidence matrices D^k, D~^k are built here by enumerating the index
triples of the output space and writing the +-1 entries of the Cartesian-grid exterior
derivative; nothing is computed in floating point.
"""
import numpy as np
import scipy.sparse as sp

from .splines import space_dim


def component_spaces(cplx, k):
    """Per-component triples (space_x, space_y, space_z) of the univariate spaces."""
    if cplx == "primal":
        P, L = "Sp", "Sp1"       # degree p (trimmed B-splines), degree p-1 (CS)
    elif cplx == "primalF":
        P, L = "SpF", "Sp1"      # the full X^k_h (untrimmed S_p), for the lifting
    elif cplx == "dual":
        P, L = "Dp1", "Dp2"      # degree p-1 (B-splines), degree p-2 (CS)
    else:
        raise ValueError(cplx)
    if k == 0:
        return [(P, P, P)]
    if k == 1:
        return [(L, P, P), (P, L, P), (P, P, L)]
    if k == 2:
        return [(P, L, L), (L, P, L), (L, L, P)]
    if k == 3:
        return [(L, L, L)]
    raise ValueError(k)


def component_shapes(cplx, k, p, n):
    """Shapes (nx, ny, nz) of each component; n = (nx_el, ny_el, nz_el)."""
    n = _n3(n)
    return [tuple(space_dim(s[a], p, n[a]) for a in range(3)) for s in component_spaces(cplx, k)]


def form_dim(cplx, k, p, n):
    return sum(int(np.prod(s)) for s in component_shapes(cplx, k, p, n))


def offsets(cplx, k, p, n):
    sh = component_shapes(cplx, k, p, n)
    off = [0]
    for s in sh:
        off.append(off[-1] + int(np.prod(s)))
    return off


def split(v, cplx, k, p, n):
    """Split a flat form vector into component arrays shaped [z][y][x]."""
    sh = component_shapes(cplx, k, p, n)
    off = offsets(cplx, k, p, n)
    return [v[off[c]:off[c + 1]].reshape(s[2], s[1], s[0]) for c, s in enumerate(sh)]


def join(comps):
    return np.concatenate([np.asarray(c).ravel() for c in comps])


def _n3(n):
    return (n, n, n) if np.isscalar(n) else tuple(n)


# --- incidence matrices ------------------------------------------------------------------------

def _deriv_terms(cplx, kout):
    """Terms (sign, input component, axis) of each output component of d: k -> k+1.

    grad:  (d u)_c = d_c u
    curl:  (d e)_1 = d_y e_3 - d_z e_2 ; (d e)_2 = d_z e_1 - d_x e_3 ; (d e)_3 = d_x e_2 - d_y e_1
    div:   (d b)   = d_x b_1 + d_y b_2 + d_z b_3
    (exterior derivative on dx, dy, dz / dy^dz, dz^dx, dx^dy proxies).
    """
    if kout == 1:
        return [[(+1, 0, 0)], [(+1, 0, 1)], [(+1, 0, 2)]]
    if kout == 2:
        return [[(+1, 2, 1), (-1, 1, 2)], [(+1, 0, 2), (-1, 2, 0)], [(+1, 1, 0), (-1, 0, 1)]]
    if kout == 3:
        return [[(+1, 0, 0), (+1, 1, 1), (+1, 2, 2)]]
    raise ValueError(kout)


def incidence(cplx, k, p, n):
    """Integer sparse matrix of d: X^k -> X^{k+1} in the given complex.

    Univariate factors (reading Z3): with the CS bases,
      primal  S_p(trimmed, dim a) -> S_{p-1} (dim b):  (du)_j = u_j - u_{j-1},  u_{-1} = u_a = 0
      dual    S_{p-1}    (dim b) -> S_{p-2} (dim a):  (dv)_j = v_{j+1} - v_j
      primalF S_p(full, dim a+2)  -> S_{p-1} (dim b):  (dU)_j = U_{j+1} - U_j  (U_0, U_{a+1}: the
              boundary functions; the trimmed rule is this one with U_0 = U_{a+1} = 0)
    """
    n = _n3(n)
    sh_in = component_shapes(cplx, k, p, n)
    sh_out = component_shapes(cplx, k + 1, p, n)
    off_in = offsets(cplx, k, p, n)
    off_out = offsets(cplx, k + 1, p, n)
    rows, cols, vals = [], [], []
    for co, terms in enumerate(_deriv_terms(cplx, k + 1)):
        so = sh_out[co]
        iz, iy, ix = np.meshgrid(np.arange(so[2]), np.arange(so[1]), np.arange(so[0]), indexing="ij")
        out_idx = off_out[co] + (ix + so[0] * (iy + so[1] * iz)).ravel()
        for sign, ci, ax in terms:
            si = sh_in[ci]
            for shift, coef in ((0, +1), (-1, -1)) if cplx == "primal" else ((+1, +1), (0, -1)):
                src = [ix.ravel().copy(), iy.ravel().copy(), iz.ravel().copy()]
                src[ax] = src[ax] + shift
                ok = (src[ax] >= 0) & (src[ax] < si[ax])
                # the two non-differentiated axes have identical extents in input and output
                in_idx = off_in[ci] + src[0] + si[0] * (src[1] + si[1] * src[2])
                rows.append(out_idx[ok])
                cols.append(in_idx[ok])
                vals.append(np.full(int(ok.sum()), sign * coef, dtype=np.int64))
    N_out, N_in = off_out[-1], off_in[-1]
    M = sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                      shape=(N_out, N_in), dtype=np.int64)
    M.sum_duplicates()
    M.eliminate_zeros()
    return M
