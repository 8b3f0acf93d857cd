#!/usr/bin/env python
"""BASELINE.json configs[4]: Kronecker wedge-solve and full-step throughput over p in {2, 3, 4} and
n_el in {32, 64, 128, 160} (identity geometry, eps = mu = 1, seeded N(0,1) right-hand sides for all
three 1-form components).  One JSON line per (p, n):
  kron_solve: x = K1^{-1} r (sgm_kron_solve: three sweeps, 48 B per element algorithmic, 16 B floor)
  step: sgm_step on a dedicated stream (graph replay), DOF-updates/s and the step's algorithmic bytes
Timing: CUDA events on the launching stream after warm-up; L2 is flushed (a 256 MB write) before
each timed repetition of the solve; the step's working set exceeds L2 from 64^3 up.
    python scripts/c5_sweep.py [--out profiles/r1_c5_sweep.jsonl]"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2302_04979_b200 as S  # noqa: E402
import synth  # noqa: E402
import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r1_c5_sweep.jsonl"))
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    peak, _ = bench.peaks()
    flush = torch.empty(32 * 1024 * 1024, dtype=torch.float64, device=dev)
    st = torch.cuda.Stream()
    lines = []
    for p in (2, 3, 4):
        for n in (32, 64, 128, 160):
            pl = S.Plan(n, p)
            N_e, N_h = pl.N_e, pl.N_h
            r = torch.from_numpy(synth.normal(7, N_e)[0]).to(dev)
            x = torch.empty_like(r)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(st):
                for _ in range(3):
                    pl.kron_solve(S.K1, r, x, stream=st)
                tot = 0.0
                for _ in range(args.reps):
                    flush.fill_(1.0)
                    a.record(st)
                    pl.kron_solve(S.K1, r, x, stream=st)
                    b.record(st)
                    st.synchronize()
                    tot += a.elapsed_time(b)
                ms_solve = tot / args.reps
                # full step (graph replay on this stream)
                d0, b0 = synth.normal(5, N_e, N_h)
                d = torch.from_numpy(d0).to(dev)
                bb = torch.from_numpy(b0).to(dev)
                e = torch.empty_like(d)
                h = torch.empty_like(bb)
                pl.hodge_star(S.MASS_EPS, d, e, stream=st)
                pl.hodge_star(S.MASS_MU, bb, h, stream=st)
                dt = 0.5 * bench.CFL_N[p] / n
                K = 50 if n >= 128 else 200
                pl.step(d, e, bb, h, dt, 5, stream=st)
                st.synchronize()
                a.record(st)
                pl.step(d, e, bb, h, dt, K, stream=st)
                b.record(st)
                st.synchronize()
                ms_step = a.elapsed_time(b) / K
            step_bytes = sum(v for _, v in bench.launch_bytes(pl, S, N_e, N_h, False))
            rec = {"p": p, "n_el": n, "N_e": N_e, "N_h": N_h,
                   "kron_solve": {"us": 1e3 * ms_solve, "algo_bytes": 48 * N_e,
                                  "gbs": 48 * N_e / (ms_solve * 1e-3) / 1e9,
                                  "frac": 48 * N_e / (ms_solve * 1e-3) / 1e9 / peak,
                                  "floor_gbs": 16 * N_e / (ms_solve * 1e-3) / 1e9},
                   "step": {"us": 1e3 * ms_step, "dof_updates_per_s": (N_e + N_h) / (ms_step * 1e-3),
                            "algo_bytes": step_bytes, "gbs": step_bytes / (ms_step * 1e-3) / 1e9,
                            "frac": step_bytes / (ms_step * 1e-3) / 1e9 / peak},
                   "peak_gbs": peak}
            lines.append(rec)
            print(json.dumps(rec), flush=True)
            pl.close()
    with open(args.out, "w") as f:
        for rec in lines:
            f.write(json.dumps(rec) + "\n")


if __name__ == "__main__":
    main()
