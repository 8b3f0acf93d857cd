"""Seeded synthetic input draws shared by the oracle tests, the GPU tests and bench.py.

This module holds NONE of the method's arithmetic: only random draws (numpy default_rng with
the per-config seeds of SURVEY 8(d): rng(k) for config Ck, draws in the listed order) and a
spectral smoothing filter used to shape a random field.  Anything that needs spline spaces,
masses, pairings or solves (projections, consistent e/h, CFL) lives in ``oracle.workloads``.
"""
import numpy as np


def rng(k):
    return np.random.default_rng(k)


def normal(k, *sizes):
    """Independent N(0,1) vectors of the given sizes from rng(k), drawn in order."""
    g = rng(k)
    return [g.standard_normal(s) for s in sizes]


def c2_amplitudes():
    """C2: alpha = rng(2).uniform(-1, 1, 4) (BASELINE.json configs[1])."""
    return rng(2).uniform(-1.0, 1.0, 4)


def c3_centres():
    """C3: inclusion centre c_eps = rng(3).uniform(.25,.75,3), then pulse centre
    c_J = rng(3).uniform(.2,.8,3) (second draw of the same generator)."""
    g = rng(3)
    c_eps = g.uniform(0.25, 0.75, 3)
    c_J = g.uniform(0.2, 0.8, 3)
    return c_eps, c_J


def smooth_field(k, shape):
    """C4 random smooth coefficients: N(0,1) from rng(k) -> orthonormal DCT-II ->
    multiply by 1/(1+|kappa|^2) (kappa = integer DCT index triple) -> inverse DCT.
    ``shape`` is [z][y][x]."""
    from scipy.fft import dctn, idctn
    g = rng(k)
    x = g.standard_normal(shape)
    X = dctn(x, norm="ortho")
    kz, ky, kx = np.meshgrid(*[np.arange(s) for s in shape], indexing="ij")
    X /= 1.0 + (kx ** 2 + ky ** 2 + kz ** 2)
    return idctn(X, norm="ortho")


def smooth_fields(k, shapes):
    """C4 initial E: one N(0,1) draw per component from ONE generator rng(k) (drawn in component
    order), each filtered like ``smooth_field``: orthonormal DCT-II -> 1/(1+|kappa|^2) -> inverse.
    ``shapes``: [z][y][x] shape of each component."""
    from scipy.fft import dctn, idctn
    g = rng(k)
    out = []
    for shape in shapes:
        x = g.standard_normal(shape)
        X = dctn(x, norm="ortho")
        kz, ky, kx = np.meshgrid(*[np.arange(s) for s in shape], indexing="ij")
        X /= 1.0 + (kx ** 2 + ky ** 2 + kz ** 2)
        out.append(idctn(X, norm="ortho"))
    return out


def gaussian_z(X, centre, sigma):
    """The C3 source potential A(x) = z-hat exp(-|x - c|^2 / (2 sigma^2)) at points X[..., 3]."""
    r2 = np.sum((np.asarray(X) - np.asarray(centre)) ** 2, axis=-1)
    A = np.zeros(np.shape(X))
    A[..., 2] = np.exp(-r2 / (2.0 * sigma ** 2))
    return A


def pulse(t, t0=0.15, width=0.05):
    """C3 source amplitude s(t) = exp(-((t - t0)/width)^2) (reading Z16)."""
    return np.exp(-((np.asarray(t) - t0) / width) ** 2)


def c3_map(X):
    """BASELINE.json configs[2] geometry, a closed-form input: x -> x + 0.1 sin(pi x) sin(pi y)
    sin(pi z) (1, 1, 1) on the unit cube (X[..., 3] -> F[..., 3])."""
    s = 0.1 * np.sin(np.pi * X[..., 0]) * np.sin(np.pi * X[..., 1]) * np.sin(np.pi * X[..., 2])
    return X + s[..., None]
