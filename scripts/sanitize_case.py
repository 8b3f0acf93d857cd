"""Small end-to-end exercise of every device entry point (for compute-sanitizer runs):
separable and general-Hodge steps with a source, kron solves (K1, K~1, transposed), pairing and
mass applies, Hodge stars, curls, energy, Gauss residuals, source check, host-buffer step."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2302_04979_b200 as S  # noqa: E402


def run(p, n, general):
    pl = S.Plan(n, p)
    if general:
        X = pl.qp_coords()
        pl.set_material(S.EPS, 1 + 0.5 * np.sin(2 * np.pi * X[:, 0]))
    g = np.random.default_rng(1)
    Ne, Nh = pl.N_e, pl.N_h
    d, e = (torch.from_numpy(g.standard_normal(Ne)).cuda() for _ in range(2))
    b, h = (torch.from_numpy(g.standard_normal(Nh)).cuda() for _ in range(2))
    a = torch.from_numpy(g.standard_normal(Nh)).cuda()
    j = torch.empty_like(d)
    pl.curl(S.CURL_DUAL, a, j)
    amp = torch.linspace(0, 1, 3, dtype=torch.float64).cuda()
    pl.step(d, e, b, h, 1e-3, 3, j_hat=j, j_amp=amp)
    for which, N in ((S.K1, Ne), (S.KT1, Nh)):
        x = torch.from_numpy(g.standard_normal(N)).cuda()
        y = torch.empty_like(x)
        for T in (False, True):
            pl.kron_solve(which, x, y, transpose=T)
            pl.pairing_apply(which, x, y, transpose=T)
    y = torch.empty_like(d)
    pl.hodge_apply(S.MASS_EPS, d, y)
    pl.hodge_star(S.MASS_EPS, d, y)
    y = torch.empty_like(b)
    pl.hodge_apply(S.MASS_MU, b, y)
    pl.hodge_star(S.MASS_MU, b, y)
    y = torch.empty_like(b)
    pl.curl(S.CURL_PRIMAL, e, y)
    out = torch.zeros(2, dtype=torch.float64).cuda()
    pl.energy(d, e, b, h, out)
    pl.gauss(d, b, out)
    assert pl.check_source(j) == 0
    hs = [x.cpu().numpy().copy() for x in (d, e, b, h)]
    pl.step_host(*hs, 1e-3, 2)
    torch.cuda.synchronize()


if __name__ == "__main__":
    for p, n, gen in ((2, 7, False), (3, (9, 6, 5), False), (4, 5, True), (3, 34, False)):
        run(p, n, gen)
    print("sanitize case ok")
