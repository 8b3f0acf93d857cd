"""CPU oracle for arXiv 2302.04979 (scheme 2 leapfrog step) -- TEST INFRASTRUCTURE ONLY.

This package is a plain, slow, obviously-correct NumPy/SciPy implementation of what the
B200 hot path computes.  It exists to prove parity; it is NOT part of the product.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import it.  The CUDA path (``paper_2302_04979_b200``) never
imports it and it never imports the CUDA path; the two share no code.  The only module both
sides use is ``synth`` (seeded random draws, none of the method's arithmetic).

Layout
------
``splines``    1D knot vectors, Cox--de Boor B-splines, Curry--Schoenberg scaling, Gauss rules
               (sec. 2.3; sec. 4.1).
``forms``      component spaces of the primal/dual complexes and the integer incidence
               matrices D^k, D~^k built by enumerating index triples.
``assemble``   tier A: 3D-quadrature assembly of the pairing matrices K1, K~1
               and of the metric/material 2-form mass matrices M~2_{1/eps}, M2_{1/mu}
                with explicit physical pull-backs.
``scheme``     tier A: scheme 2 (eqs. discrete2_*) with a generic sparse direct
               solve (SuperLU) per Kronecker block; energy and Gauss residuals.
``structured`` tier B: the same step via the paper's own Kronecker identities
               (eq. kroninverse, vec trick P:L575-585) with dense 1D inverses and
               sum-factorised mass applies; pinned against tier A.
``workloads``  closed-form cavity modes, L2 projections of initial data, CFL power iteration,
               and the BASELINE.json configs C1-C5.

Parity status: every function is pinned in ``tests/test_oracle_*.py`` against facts the paper
and mathematics fix (closed forms, identities, invariants, brute force on tiny grids).
The single documented exception is the CFL estimate (``workloads.cfl_dt_max``): its absolute
value is "parity unpinned" (DESIGN.md readings), only its p- and h-scalings are pinned.
"""
