"""Run a matrix of sweep configurations through the library the binding loads (the product build,
or the verification build with SGM_LIB_VARIANT=checked: csrc/check.cuh) and save every result.

Each case exercises the pipelined sweeps in one launch configuration: degrees 2-4, strided and
x-line (bulk and line-by-line bulk) passes, 32- and 64-line tiles (SGM_OPT_WIDE_TILES), ragged last tiles, several work items per CTA (slab
reuse), long lines (many consumer warps, truncated SPIKE reach), the schedules (reduced, full,
serial, fused, exact spikes), the general Hodge path, the (e,h)-state step and the Kronecker
solves.  Used by tests/test_gpu_checked.py:

    python scripts/checked_cases.py OUT.npz [--reps R] [--cases a,b,...]

writes OUT.npz (one array per case: the first repetition's result) and prints one JSON line
{"variant", "cases": {name: {"violations", "first", "reps_identical", "finite"}}}.
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2302_04979_b200 as S  # noqa: E402

# name -> (degree, n_el, options, kind)
CASES = {
    "p2_ragged": (2, (20, 21, 22), 0, "step"),
    "p3_ragged": (3, (33, 17, 40), 0, "step"),
    "p4_ragged": (4, (24, 30, 19), 0, "step"),
    "p2_ragged_wide": (2, (20, 21, 22), S.OPT_WIDE_TILES, "step"),
    "p3_ragged_wide": (3, (33, 17, 40), S.OPT_WIDE_TILES, "step"),
    "p4_ragged_wide": (4, (24, 30, 19), S.OPT_WIDE_TILES | S.OPT_FULL_SCHEDULE, "step"),
    "p3_128": (3, (128, 128, 128), 0, "step"),
    "p2_96_serial": (2, (96, 96, 96), S.OPT_SERIAL, "step"),
    "p3_full": (3, (64, 48, 40), S.OPT_FULL_SCHEDULE, "step"),
    "p3_fused": (3, (64, 48, 40), S.OPT_FUSED, "step"),
    "p4_fused_full": (4, (40, 44, 36), S.OPT_FUSED | S.OPT_FULL_SCHEDULE, "step"),
    "p3_exact_spike": (3, (150, 40, 36), S.OPT_EXACT_SPIKE, "step"),
    "p2_long_x": (2, (300, 16, 20), 0, "step"),
    "p4_max_line": (4, (389, 8, 9), 0, "step"),
    "p3_general": (3, (24, 20, 18), 0, "general"),
    "p3_eh": (3, (32, 33, 34), 0, "eh"),
    "p3_eh_fused": (3, (32, 33, 34), S.OPT_FUSED, "eh"),
    "p4_kron": (4, (50, 41, 37), 0, "kron"),
}


def run_case(p, n, opts, kind):
    pl = S.Plan(n, p)
    pl.set_options(opts)
    g = np.random.default_rng(7)
    Ne, Nh = pl.N_e, pl.N_h
    if kind == "general":
        X = pl.qp_coords()
        pl.set_material(S.EPS, 1 + 0.5 * np.sin(2 * np.pi * X[:, 0]) * np.cos(np.pi * X[:, 2]))
    d, e = (torch.from_numpy(g.standard_normal(Ne)).cuda() for _ in range(2))
    b, h = (torch.from_numpy(g.standard_normal(Nh)).cuda() for _ in range(2))
    a = torch.from_numpy(g.standard_normal(Nh)).cuda()
    j = torch.empty_like(d)
    pl.curl(S.CURL_DUAL, a, j)
    amp = torch.linspace(0.2, 1, 4, dtype=torch.float64).cuda()
    dt = 1e-3
    if kind in ("step", "general"):
        pl.step(d, e, b, h, dt, 4, j_hat=j, j_amp=amp)
        out = [d, e, b, h]
    elif kind == "eh":
        pl.step_eh(e, h, dt, 4, j_hat=j, j_amp=amp)
        out = [e, h]
    else:
        out = []
        for which, N in ((S.K1, Ne), (S.KT1, Nh)):
            x = torch.from_numpy(g.standard_normal(N)).cuda()
            for T in (False, True):
                y = torch.empty_like(x)
                pl.kron_solve(which, x, y, transpose=T)
                out.append(y)
    torch.cuda.synchronize()
    r = torch.cat([o.flatten() for o in out]).cpu().numpy()
    pl.close()
    return r


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("out")
    ap.add_argument("--reps", type=int, default=1)
    ap.add_argument("--cases", default="")
    a = ap.parse_args()
    names = [c for c in a.cases.split(",") if c] or list(CASES)
    checked = S.VARIANT == "checked"
    res, summ = {}, {}
    for name in names:
        p, n, opts, kind = CASES[name]
        if checked:
            S.check_read(reset=True)
        first = run_case(p, n, opts, kind)
        same = True
        for _ in range(a.reps - 1):
            same &= bool(np.array_equal(first, run_case(p, n, opts, kind)))
        viol, code = S.check_read(reset=True) if checked else (0, 0)
        res[name] = first
        summ[name] = {"violations": viol, "first": code, "reps_identical": same,
                      "finite": bool(np.isfinite(first).all())}
    np.savez(a.out, **res)
    print(json.dumps({"variant": S.VARIANT or "product", "version": S.sgm_version().decode(), "cases": summ}))


if __name__ == "__main__":
    main()
