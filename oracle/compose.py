"""Higher-order time integration by symmetric composition of leapfrog sub-steps
(TEST INFRASTRUCTURE ONLY).

The paper names "higher-order symplectic time integrators" as future work; SURVEY 8(f)
NEXT #4 builds them by composing the scheme-2 leapfrog.  Reading Z25: the sub-step is
the kick-drift-kick (velocity Verlet) form of eqs. discrete2_* with b synchronous,
    S(tau):  b <- b - (tau/2) D1 e;  h = K~1^{-1} M2 b
             d <- d + tau (D~1 h - s j^);  e = K1^{-1} M~2 d
             b <- b - (tau/2) D1 e;  h = K~1^{-1} M2 b
and one step of size dt is S(w_0 dt) ... S(w_{m-1} dt).  Yoshida's triple jump (Yoshida 1990,
"Construction of higher order symplectic integrators"): w = (x1, x0, x1) with
x1 = 1/(2 - 2^{1/3}), x0 = -2^{1/3}/(2 - 2^{1/3}) gives 4th order because the sub-step is
symmetric and 2 x1^3 + x0^3 = 0, 2 x1 + x0 = 1.

Written step by step without merging adjacent kicks (the CUDA path merges them).  Pinned in
tests/test_oracle_scheme.py: w = (1,) against the staggered leapfrog, and the time order against
the exact solution of the semi-discrete system (matrix exponential of the dense tier-A operator).
"""
import numpy as np

from .workloads import _ops

_C = 2.0 ** (1.0 / 3.0)
YOSHIDA4 = (1.0 / (2.0 - _C), -_C / (2.0 - _C), 1.0 / (2.0 - _C))


def kdk(tb, d, e, b, h, tau, jhat=None, s=1.0):
    """One kick-drift-kick sub-step S(tau) on flat vectors (tier A or tier B `tb`)."""
    hodge_eps, hodge_mu, _, _, D1, Dt1 = _ops(tb)
    b = b - 0.5 * tau * D1(e)
    h = hodge_mu(b)
    if jhat is not None:
        d = d + tau * (Dt1(h) - s * jhat)
    else:
        d = d + tau * Dt1(h)
    e = hodge_eps(d)
    b = b - 0.5 * tau * D1(e)
    h = hodge_mu(b)
    return d, e, b, h


def run_composed(tb, d, e, b, h, dt, n_steps, weights=YOSHIDA4, jhat=None, jamp=None):
    """n_steps composed steps; jamp[k*m + i] is s for sub-step i of step k (None -> 1)."""
    m = len(weights)
    for k in range(n_steps):
        for i, wi in enumerate(weights):
            s = 1.0 if jamp is None else jamp[k * m + i]
            d, e, b, h = kdk(tb, d, e, b, h, wi * dt, jhat, s)
    return d, e, b, h
