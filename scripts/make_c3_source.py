#!/usr/bin/env python
"""Writes tests/golden/c3_a_hat.npz: the C3 source potential a^ (configs[2]; reading Z16/Z28), the
unweighted parametric L2 projection onto X~1 of z-hat exp(-|F(x^) - c_J|^2 / (2 0.05^2)) at 48^3,
p = 3, from the oracle (oracle.workloads).  bench.py reads it to build j^ = D~1 a^ with the library's
curl (the bench never executes the oracle).  Usage: python scripts/make_c3_source.py"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402
from oracle import workloads as W  # noqa: E402


def main(p=3, n=48):
    ctrl, _, _ = W.c3_setup(p, n)
    _, c_J = synth.c3_centres()
    a = W.project_dual1(p, n, synth.gaussian_z(W.physical_points(p, n, ctrl), c_J, W.C3_SIGMA))
    out = os.path.join(ROOT, "tests", "golden", "c3_a_hat.npz")
    np.savez_compressed(out, a_hat=a, p=p, n=n,
                        source="scripts/make_c3_source.py (oracle.workloads.project_dual1, reading Z28)")
    print(out, a.shape, os.path.getsize(out))


if __name__ == "__main__":
    main()
