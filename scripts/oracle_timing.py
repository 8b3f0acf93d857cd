#!/usr/bin/env python
"""CPU oracle timing beside the GPU: the oracle as it stands, per step, on this host's
cores, for the BASELINE.json configurations -- tier A (assembled matrices, SuperLU) for C1 where it
is feasible, tier B (Kronecker) for every config.  Setup (assembly, factorisation) is excluded;
1 warm-up step, then the median of >= 3 timed steps (bounded by --budget seconds per config).

    python scripts/oracle_timing.py [--out profiles/r1_cpu_oracle.jsonl] [--budget 20]"""
import argparse
import json
import os
import platform
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from oracle import forms  # noqa: E402
from oracle import workloads as W  # noqa: E402
from oracle.assemble import Quad, physical_qp  # noqa: E402
from oracle.scheme import TierA  # noqa: E402
from oracle.structured import TierB  # noqa: E402


def time_steps(step, st, budget):
    st = step(st)  # warm-up
    ts = []
    t_end = time.perf_counter() + budget
    while len(ts) < 3 or (time.perf_counter() < t_end and len(ts) < 20):
        t0 = time.perf_counter()
        st = step(st)
        ts.append(time.perf_counter() - t0)
    return float(np.median(ts)), len(ts)


def configs():
    yield "C1 cavity p=2 8^3 (tier A)", 2, 8, "A", None, None
    yield "C1 cavity p=2 8^3", 2, 8, "B", None, None
    yield "C2 p=3 32^3", 3, 32, "B", None, None
    yield "C3 curved p=3 48^3, eps inclusion", 3, 48, "B", "c3", "c3"
    yield "C4 p=4 96^3, variable eps", 4, 96, "B", None, "c4"
    for p in (2, 3, 4):
        for n in (32, 64, 128, 160):
            yield f"C5 p={p} {n}^3", p, n, "B", None, None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r1_cpu_oracle.jsonl"))
    ap.add_argument("--budget", type=float, default=20.0)
    args = ap.parse_args()
    import threadpoolctl
    recs = []
    for name, p, n, tier, geo, mat in configs():
        ctrl = W.interpolate_map(p, n, W.c3_map) if geo == "c3" else None
        inv_eps = 1.0
        if mat is not None:
            X = physical_qp(Quad(p, n), ctrl).reshape(-1, 3)
            if mat == "c3":
                c_eps, _ = synth.c3_centres()
                inv_eps = 1.0 / np.where(np.linalg.norm(X - c_eps, axis=1) < 0.25, 4.0, 1.0)
            else:
                inv_eps = 1.0 / (1 + 0.5 * np.sin(2 * np.pi * X[:, 0]) * np.cos(2 * np.pi * X[:, 1]))
        t0 = time.perf_counter()
        if tier == "A":
            tb = TierA(p, n)
        else:
            tb = TierB(p, n, ctrl=ctrl, inv_eps=inv_eps, inv_mu=1.0)
        setup = time.perf_counter() - t0
        d0, b0 = synth.normal(5, tb.N_e, tb.N_h)
        dt = 0.1 / n
        st = (d0, d0.copy(), b0, b0.copy())
        med, k = time_steps(lambda s: tb.step(*s, dt), st, args.budget)
        threads = max([i.get("num_threads", 1) for i in threadpoolctl.threadpool_info()] + [1])
        rec = {"config": name, "tier": tier, "p": p, "n_el": n, "dofs": tb.N_e + tb.N_h,
               "s_per_step": med, "steps_timed": k, "dof_updates_per_s": (tb.N_e + tb.N_h) / med,
               "setup_s": setup, "cores": os.cpu_count(), "blas_threads": threads,
               "cpu": platform.processor() or platform.machine(),
               "note": "tier A: SuperLU (single-threaded) per Kronecker block" if tier == "A" else
                       "tier B: dense 1D inverses / sum factorisation via NumPy BLAS"}
        recs.append(rec)
        print(json.dumps(rec), flush=True)
    with open(args.out, "w") as f:
        for r in recs:
            f.write(json.dumps(r) + "\n")


if __name__ == "__main__":
    main()
