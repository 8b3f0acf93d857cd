#!/usr/bin/env python
"""Writes tests/golden/workload_dt.json: dt = 0.5 * dt_max for the BASELINE configs C1-C4, with
dt_max = 2 / sqrt(lambda_max) of each config's own scheme-2 leapfrog operator by the oracle's power
iteration (SURVEY 8(d) "Fixing dt reproducibly": start vector rng(100 + k), 300 iterations, Rayleigh
quotient; reading Z15).  Calls only oracle/ (and synth/ for the seeded draws); 17 significant
digits.  Usage: python scripts/make_workload_dt.py [c1 c2 c3 c4]"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402
from oracle import workloads as W  # noqa: E402
from oracle.structured import TierB  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "workload_dt.json")


def operator(cfg):
    if cfg == "c1":
        return 1, TierB(2, 8)
    if cfg == "c2":
        return 2, TierB(3, 32)
    if cfg == "c3":
        ctrl, eps, _ = W.c3_setup(3, 48)
        return 3, TierB(3, 48, ctrl=ctrl, inv_eps=1.0 / eps, inv_mu=1.0)
    eps, tb = W.c4_setup(4, 96)
    return 4, tb


def main(cfgs):
    out = json.load(open(OUT)) if os.path.exists(OUT) else {}
    out["_source"] = ("scripts/make_workload_dt.py: dt = 0.5 * 2/sqrt(lambda), lambda = oracle "
                      "workloads.cfl_power (300 iterations from rng(100 + k)) of each config's own operator")
    for cfg in cfgs:
        t0 = time.time()
        k, tb = operator(cfg)
        if cfg == "c3":   # tier B keeps a separable mu only for the identity map
            tb.sep_mu = None
            tb.W_mu = tb._W(1.0)
        x0 = synth.rng(100 + k).standard_normal(tb.N_e)
        lam, dtmax, _, lams = W.cfl_power(tb, x0, 300)
        out[cfg] = {"dt": float(f"{0.5 * dtmax:.17g}"), "dt_max": float(f"{dtmax:.17g}"),
                    "lambda": float(f"{lam:.17g}"), "lambda_prev": float(f"{lams[-2]:.17g}"),
                    "seconds": round(time.time() - t0, 1)}
        print(cfg, out[cfg], flush=True)
        json.dump(out, open(OUT, "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1:] or ["c1", "c2", "c3", "c4"])
