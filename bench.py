#!/usr/bin/env python
"""Benchmark of one scheme-2 leapfrog step (arXiv 2302.04979) on B200.

Metric (BASELINE.json): fp64 DOF-updates/s per leapfrog step, DOF-updates = (N_e + N_h) per
step, and the HBM-roofline fraction of the dominant kernel.  Default workload: configs[4] (C5)
full step at p = 3, 128^3 elements, identity geometry, eps = mu = 1 -- the configuration the
north-star target (>= 60 % of HBM roofline) is stated on.  Inputs: seeded N(0,1) d, b (rng(5)),
e, h derived by the discrete Hodge stars on the device (setup, untimed).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c5 --p 3 --n 128]

Multi-GPU (torchrun): the path does not shard (north_star: one GPU, no collectives), so every
rank runs an independent replica ("replicas only", scaling "weak"); the only collective is the
max-over-ranks of the device-timed region.
"""
import argparse
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fp64 DOF-updates/sec per leapfrog step and % of B200 HBM roofline"
UNIT = "DOF-updates/s"
# Delta t_max * n for scheme 2 on the unit cube (reading Z15 -- the oracle's CFL
# routine reproduces these; used only to pick a stable dt for throughput runs)
CFL_N = {2: 0.3046, 3: 0.2020, 4: 0.1205}


def max_over_ranks(ms, dist, device):
    """Device-timed milliseconds of this rank -> max over all ranks (replicas run concurrently)."""
    if dist is None:
        return ms
    import torch
    t = torch.tensor([ms], device=device, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def aggregate_value(dofs_per_step, steps, ms_max, world):
    """Whole-job DOF-updates/s: every rank advances its own replica by `steps` steps."""
    return world * dofs_per_step * steps / (ms_max * 1e-3)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c5", choices=["c2", "c3", "c4", "c5"])
    ap.add_argument("--p", type=int, default=3)
    ap.add_argument("--n", type=int, default=128)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-variants", action="store_true", help="skip the schedule-variant timings")
    ap.add_argument("--opts", type=lambda v: int(v, 0), default=0,
                    help="SGM_OPT_* schedule option bits (0 = the production schedule)")
    ap.add_argument("--scheme", type=int, default=2, choices=[1, 2],
                    help="Hodge stars: 2 = pairing solves (the paper's method, default), 1 = mass solves")
    return ap.parse_args()


def workload(args):
    """(p, n, description, geometry ctrl or None, eps at qp or None, has_source)."""
    p, n, desc, geo, mat, src = _workload(args)
    if getattr(args, "scheme", 2) == 1:
        desc += ", scheme 1 (mass-matrix Hodge stars)"
    return p, n, desc, geo, mat, src


def _workload(args):
    if args.config == "c5":
        return args.p, args.n, f"C5 full step p={args.p} n_el={args.n}^3 identity eps=mu=1", None, None, False
    if args.config == "c2":
        return 3, 32, "C2 full step p=3 n_el=32^3 identity eps=mu=1", None, None, False
    if args.config == "c3":
        return (3, 48, "C3 full step p=3 n_el=48^3 curved map, eps in {1,4} inclusion, projected Gaussian J "
                "with Gaussian pulse s(t), zero initial fields", "c3", "c3", True)
    return (4, 96, "C4 full step p=4 n_el=96^3 identity, eps=1+0.5 sin(2pi x)cos(2pi y), smooth random E",
            None, "c4", False)


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(path))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, torch copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


def peaks_sm_mhz():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["sm_max_mhz"])
    except Exception:
        return 1965.0


class ClockSampler:
    """NVML samples of SM clock and throttle reasons while running."""

    def __init__(self, dev_index):
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self._stop = threading.Event()
        try:
            import pynvml as N
            N.nvmlInit()
            self.N = N
            self.h = N.nvmlDeviceGetHandleByIndex(dev_index)
            self.max_mhz = N.nvmlDeviceGetMaxClockInfo(self.h, N.NVML_CLOCK_SM)
        except Exception:
            self.N = None

    def _run(self):
        N = self.N
        names = {
            "hw_slowdown": getattr(N, "nvmlClocksThrottleReasonHwSlowdown", 0x8),
            "sw_thermal_slowdown": getattr(N, "nvmlClocksThrottleReasonSwThermalSlowdown", 0x20),
            "hw_thermal_slowdown": getattr(N, "nvmlClocksThrottleReasonHwThermalSlowdown", 0x40),
            "sw_power_cap": getattr(N, "nvmlClocksThrottleReasonSwPowerCap", 0x4),
            "hw_power_brake": getattr(N, "nvmlClocksThrottleReasonHwPowerBrakeSlowdown", 0x80),
        }
        while not self._stop.is_set():
            try:
                self.samples.append(N.nvmlDeviceGetClockInfo(self.h, N.NVML_CLOCK_SM))
                r = N.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                for k, v in names.items():
                    if r & v:
                        self.reasons.add(k)
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.N is not None:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.N is not None:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def device_cfl(pl, S, torch, dev, seed, n_iter=300):
    """dt_max of the plan's own scheme-2 operator by the library's power iteration (sgm_cfl; SURVEY
    8(d): start vector rng(100 + k), 300 iterations, Rayleigh quotient; reading Z15)."""
    import synth
    x = torch.from_numpy(synth.rng(seed).standard_normal(pl.N_e)).to(dev)
    e = torch.empty(pl.N_e, dtype=torch.float64, device=dev)
    b = torch.empty(pl.N_h, dtype=torch.float64, device=dev)
    h = torch.empty_like(b)
    out = torch.zeros(2, dtype=torch.float64, device=dev)
    pl.cfl(x, e, b, h, out, n_iter)
    return float(out[1].item())


def build_inputs(args, torch, S, dev):
    """The configured workloads (BASELINE.json configs) built with
    the library and synth only (the bench never executes the oracle outside its CPU legs):
      C5 / C2: d0, b^{1/2} ~ N(0,1) (rng(5)), e0, h^{1/2} by the discrete Hodge stars;
      C3: the curved map (library Greville interpolation), eps in {1, 4} inclusion, ZERO initial
          fields, j^ = D~1 a^ with a^ the oracle-written projected Gaussian (tests/golden/c3_a_hat.npz,
          scripts/make_c3_source.py), s(t) = exp(-((t - 0.15)/0.05)^2), dt = 0.5 dt_max (sgm_cfl);
      C4: eps = 1 + 0.5 sin(2 pi x) cos(2 pi y), e0 = the smoothed rng(4) field (synth.smooth_fields),
          d0 = K1 e0 (the parity tests use d0 = M~2^{-1} K1 e0 by PCG: same smoothness class, one mass
          solve fewer, throughput unaffected), e0 = K1^{-1} M~2 d0, b^{1/2} = -(dt/2) D1 e0,
          h^{1/2} = K~1^{-1} M2 b^{1/2}; dt = 0.5 dt_max (sgm_cfl)."""
    import synth
    p, n, desc, geo, mat, src = workload(args)
    ctrl = None
    if geo == "c3":
        # the closed-form C3 map interpolated at the Greville points by the library (reading Z18)
        ctrl = S.interpolate_geometry(n, p, synth.c3_map)
    pl = S.Plan(n, p, geom_ctrl=ctrl, device=dev.index or 0)
    if getattr(args, "scheme", 2) == 1:
        pl.set_scheme(1)
    pl.set_options(getattr(args, "opts", 0))
    if mat is not None:
        X = pl.qp_coords()
        if mat == "c3":
            c_eps, _ = synth.c3_centres()
            eps = np.where(np.linalg.norm(X - c_eps, axis=1) < 0.25, 4.0, 1.0)
        else:
            eps = 1 + 0.5 * np.sin(2 * np.pi * X[:, 0]) * np.cos(2 * np.pi * X[:, 1])
        pl.set_material(S.EPS, eps)
        del X
    jhat = None
    if args.config == "c3":
        dt = 0.5 * device_cfl(pl, S, torch, dev, 103)
        a = np.load(os.path.join(ROOT, "tests", "golden", "c3_a_hat.npz"))["a_hat"]
        jhat = torch.empty(pl.N_e, dtype=torch.float64, device=dev)
        pl.curl(S.CURL_DUAL, torch.from_numpy(a).to(dev), jhat)   # j = D~1 a: divergence free
        z = [torch.zeros(k, dtype=torch.float64, device=dev) for k in (pl.N_e, pl.N_e, pl.N_h, pl.N_h)]
        d, e, b, h = z
    elif args.config == "c4":
        dt = 0.5 * device_cfl(pl, S, torch, dev, 104)
        shapes = [tuple(pl.shape(S.FORM_E, c)[::-1]) for c in range(3)]
        e0 = torch.from_numpy(np.concatenate([f.ravel() for f in synth.smooth_fields(4, shapes)])).to(dev)
        d = torch.empty_like(e0)
        pl.pairing_apply(S.K1, e0, d)
        e = torch.empty_like(d)
        pl.hodge_star(S.MASS_EPS, d, e)
        b = torch.empty(pl.N_h, dtype=torch.float64, device=dev)
        pl.curl(S.CURL_PRIMAL, e, b)
        b.mul_(-0.5 * dt)
        h = torch.empty_like(b)
        pl.hodge_star(S.MASS_MU, b, h)
    else:
        d0, b0 = synth.normal(5, pl.N_e, pl.N_h)
        d = torch.from_numpy(d0).to(dev)
        b = torch.from_numpy(b0).to(dev)
        e = torch.empty_like(d)
        h = torch.empty_like(b)
        pl.hodge_star(S.MASS_EPS, d, e)
        pl.hodge_star(S.MASS_MU, b, h)
        dt = 0.5 * CFL_N[p] / n
    torch.cuda.synchronize()
    return pl, (d, e, b, h), jhat, dt, desc, p, n


def launch_bytes(pl, S, N_e, N_h, has_src):
    """Algorithmic bytes of every kernel launch of one step, in launch order: [(class, bytes)].
    A sweep reads its input form and writes its output form once (16 B per element); the update
    reads the curl source, the state (and j^) and writes the state; the general Hodge reads x and the
    quadrature weights W and read-modify-writes y ("Kernels and their rooflines")."""
    out = []
    mode = pl.schedule_mode()
    for half, (N, Ns, pre) in enumerate(((N_e, N_h, "eps"), (N_h, N_e, "mu"))):
        src = 8 * N if (half == 0 and has_src) else 0
        sep = pl.separable(S.MASS_EPS if half == 0 else S.MASS_MU)
        if sep and (mode == 3 or (mode == 0 and pl.options() & S.OPT_FUSED)):
            # fused schedule: the update runs inside the first sweep launch, which reads the curl
            # source (N_s) and the state (N) and writes the state and the sweep output (2 N)
            out.append(("fused_" + pre, 8 * (Ns + 3 * N) + src))
            if mode == 3:
                if half == 0:  # {0 along y} || {1, 2 along x}
                    out += [("eps_y", 16 * N / 3), ("eps_x", 16 * N * 2 / 3)]
            else:
                out += [(pre + "_y", 16 * N), (pre + "_x", 16 * N)]
            continue
        out.append(("update", 8 * (Ns + 2 * N) + src))
        if sep:
            # reduced schedule: an eps pass sweeps 2 of the 3 (equal-size) components, a mu pass 1
            if not pl.reduced_schedule():
                out += [(pre + "_z", 16 * N), (pre + "_y", 16 * N), (pre + "_x", 16 * N)]
            elif half == 0 and mode == 2:
                # eps: {0 z, 1 z, 2 y} in one launch, then {0 y} and {1 x, 2 x} concurrently
                out += [(pre + "_z", 16 * N), (pre + "_y", 16 * N / 3), (pre + "_x", 16 * N * 2 / 3)]
            elif half == 0:
                out += [(pre + "_z", 16 * N * 2 / 3), (pre + "_y", 16 * N * 2 / 3), (pre + "_x", 16 * N * 2 / 3)]
            else:
                out += [(pre + "_z", 16 * N * 2 / 3), (pre + "_x", 16 * N / 3)]
        else:
            wq = pl.qp_count() * (6 if pl.geom else 1) * 8
            out += [("hodge_general", 24 * N + wq), ("solve_z", 16 * N), (pre + "_y", 16 * N), (pre + "_x", 16 * N)]
    return out


def hodge_flops(pl, S, p, n):
    """Algorithmic fp64 FLOPs of one general Hodge apply per mass [(eps), (mu)] (None if separable):
    element-wise sum factorisation (per component: interpolate x -> y -> z, test back, 2 FLOPs per
    FMA) plus the quadrature-point multiply (6 FLOPs per point scalar, 15 for the full 3x3 W)."""
    Q = p + 1
    out = []
    for m, dual in ((S.MASS_EPS, True), (S.MASS_MU, False)):
        if pl.separable(m):
            out.append(None)
            continue
        fma = 0
        for c in range(3):
            k = [(p if dual else p + 1) if a == c else (p - 1 if dual else p) for a in range(3)]
            fma += 2 * (Q * k[0] * k[1] * k[2] + Q * Q * k[1] * k[2] + Q ** 3 * k[2])
        out.append(float(n) ** 3 * (2 * fma + (15 if pl.geom else 6) * Q ** 3))
    return out


def fp64_peak():
    """The measured fp64 peak (profiles/r2_fp64_peak.json, scripts/fp64_peak.py: the larger of a
    DFMA-chain kernel and cuBLAS DGEMM), else the derived 148 SMs x 64 DFMA lanes/SM/cycle x 2 FLOPs
    x max clock."""
    path = os.path.join(ROOT, "profiles", "r2_fp64_peak.json")
    try:
        d = json.load(open(path))
        v = max(float(d["dfma"]["tflops"]), float(d["dgemm_tflops"]))
        return v, "measured (profiles/r2_fp64_peak.json: max of a DFMA-chain kernel and cuBLAS DGEMM 8192^3)"
    except Exception:
        return 148 * 64 * 2 * peaks_sm_mhz() * 1e6 / 1e12, "derived: 148 SMs x 64 DFMA/SM/cycle x 2 x max SM clock"


def oracle_workload(args):
    """The CPU legs' workload (the oracle's tier B, as it stands): (tier B, state, dt, j^, amplitude
    function k -> s_k, description).  C3 / C4 follow the same recipes as the GPU inputs of
    build_inputs (C3: zero fields, projected Gaussian source, pulse; C4: smooth e0 with d0 = K1 e0)."""
    import synth
    from oracle import forms
    from oracle import workloads as Wk
    from oracle.structured import TierB, TierB1, curl_primal
    p, n, desc, geo, mat, src = workload(args)
    dts = {}
    gpath = os.path.join(ROOT, "tests", "golden", "workload_dt.json")
    if os.path.exists(gpath):
        dts = json.load(open(gpath))
    if args.config == "c3":
        ctrl, eps, _ = Wk.c3_setup(p, n)
        tb = TierB(p, n, ctrl=ctrl, inv_eps=1.0 / eps, inv_mu=1.0)
        dt = dts.get("c3", {}).get("dt", 0.25 * CFL_N[p] / n)
        jhat = Wk.c3_source(p, n, ctrl)
        st = tuple(np.zeros(k) for k in (tb.N_e, tb.N_e, tb.N_h, tb.N_h))
        return tb, st, dt, jhat, (lambda k: float(synth.pulse((k + 0.5) * dt))), desc
    if args.config == "c4":
        eps, tb = Wk.c4_setup(p, n)
        dt = dts.get("c4", {}).get("dt", 0.25 * CFL_N[p] / n)
        shapes = [tuple(s[::-1]) for s in tb.sh_e]
        e0 = forms.join(synth.smooth_fields(4, shapes))
        d0 = forms.join(tb.apply_K1(tb.split_e(e0)))
        e0 = tb.hodge_eps(d0)
        bh = -0.5 * dt * forms.join(curl_primal(tb.split_e(e0)))
        return tb, (d0, e0, bh, tb.hodge_mu(bh)), dt, None, (lambda k: 1.0), desc
    tb = TierB(p, n) if getattr(args, "scheme", 2) == 2 else TierB1(p, n)
    d0, b0 = synth.normal(5, tb.N_e, tb.N_h)
    st = (d0, tb.hodge_eps(d0), b0, tb.hodge_mu(b0))
    return tb, st, 0.5 * CFL_N[p] / n, None, (lambda k: 1.0), desc


def _threads():
    import threadpoolctl
    return max([i.get("num_threads", 1) for i in threadpoolctl.threadpool_info()] + [1])


def cpu_baseline(args, budget_s=10.0):
    """The oracle (tier B, as it stands) on this host: a bounded sample of the same workload."""
    tb, st, dt, jhat, amp, desc = oracle_workload(args)
    st = tb.step(*st, dt, jhat, amp(0))  # warm-up
    t0 = time.perf_counter()
    k = 0
    while True:
        st = tb.step(*st, dt, jhat, amp(k + 1))
        k += 1
        if time.perf_counter() - t0 > budget_s and k >= 2:
            break
    t = time.perf_counter() - t0
    return {"value": (tb.N_e + tb.N_h) * k / t, "unit": UNIT, "cores": int(_threads()), "kind": "oracle",
            "sample": f"{k} tier-B oracle steps (setup excluded) of {desc}, {t:.1f} s",
            "host_cpus": os.cpu_count()}


def run_reference(args, rank, world):
    """--impl reference: the CPU oracle timed on the host cores (rank 0 only)."""
    if rank != 0:
        return
    tb, st, dt, jhat, amp, desc = oracle_workload(args)
    p, n = tb.p, tb.n[0]
    for i in range(max(1, min(args.warmup, 2))):
        st = tb.step(*st, dt, jhat, amp(i))
    budget = 120.0
    t0 = time.perf_counter()
    k = 0
    while k < args.steps:
        st = tb.step(*st, dt, jhat, amp(k))
        k += 1
        if time.perf_counter() - t0 > budget:
            break
    t = time.perf_counter() - t0
    v = (tb.N_e + tb.N_h) * k / t
    out = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": k, "warmup": args.warmup,
           "ms_per_step": 1e3 * t / k, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
           "dtype": "f64", "data": "synthetic", "impl": "reference",
           "config": {"workload": desc, "p": p, "n_el": n, "dofs_per_step": tb.N_e + tb.N_h},
           "cpu_baseline": {"value": v, "unit": UNIT, "cores": int(_threads()), "kind": "oracle",
                            "sample": f"{k} of {args.steps} requested tier-B oracle steps (120 s cap), setup excluded"},
           "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out))


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    import torch
    import paper_2302_04979_b200 as S
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)

    pl, state, jhat, dt, desc, p, n = build_inputs(args, torch, S, dev)
    N_e, N_h = pl.N_e, pl.N_h
    dofs = N_e + N_h
    K, W = args.steps, max(3, args.warmup)
    jamp = None
    if jhat is not None:
        import synth
        jamp = torch.from_numpy(synth.pulse((np.arange(K + W) + 0.5) * dt)).to(dev)   # s(t_{k+1/2})
    stream = torch.cuda.Stream()          # a dedicated stream (sgm_step graph-captures its launches)
    torch.cuda.set_stream(stream)

    def steps(k0, k):
        # one C-ABI call for k steps (the library loops on the device stream)
        pl.step(*state, dt, k, j_hat=jhat, j_amp=None if jamp is None else jamp[k0:k0 + k], stream=stream)

    steps(0, W)
    torch.cuda.synchronize()

    def timed(profile):
        pl.set_profiling(profile)
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        steps(W, K)
        e1.record(stream)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        ms = e0.elapsed_time(e1)
        prof = pl.profile() if profile else None
        pl.set_profiling(False)
        return ms, prof

    with ClockSampler(local) as clk:
        ms, _ = timed(False)
        ms_prof, prof = timed(True)
    ms = max_over_ranks(ms, dist, dev)
    value = aggregate_value(dofs, K, ms, world)

    # ---- rooflines per kernel FUNCTION (profiled pass of the same K steps, CUDA events on the
    # launching stream around every launch).  Sweep launches of all classes are one function
    # (sweep_kernel / fsweep_kernel); concurrent launches (a fork/join pair) count once, by the longer
    # side, so the function's time is the wall time of its phases in the step.
    peak, peak_src = peaks()
    lb = launch_bytes(pl, S, N_e, N_h, jhat is not None)
    step_bytes = sum(b for _, b in lb)
    per_cls = {}
    for cls, b in lb:
        per_cls.setdefault(cls, []).append(b)
    kernels = {}
    for cls, (kms, cnt) in prof.items():
        per = kms / cnt
        kernels[cls] = {"launches": cnt, "ms_per_launch": per}
        if cls in per_cls:
            by = sum(per_cls[cls]) / len(per_cls[cls])
            kernels[cls]["algo_bytes"] = by
            kernels[cls]["gbs"] = by / (per * 1e-3) / 1e9
    mode = pl.schedule_mode()
    pairs = [("eps_y", "eps_x"), ("mu_z", "mu_x")] if mode in (2, 3) else []

    def phase_ms(classes):
        """per-step wall milliseconds of these classes (concurrent pairs by their longer side)"""
        t, seen = 0.0, set()
        for a, b in pairs:
            if a in classes and b in classes and a in prof and b in prof:
                t += max(prof[a][0], prof[b][0]) / K
                seen |= {a, b}
        return t + sum(prof[c][0] / K for c in classes if c in prof and c not in seen)

    funcs = {"sweep": [c for c in prof if c.endswith(("_z", "_y", "_x")) or c.startswith("fused_")],
             "update": [c for c in prof if c == "update"],
             "hodge_general": [c for c in prof if c == "hodge_general"]}
    step_phase = phase_ms(list(prof))
    func = {}
    for name, cls in funcs.items():
        if not cls:
            continue
        t = phase_ms(cls)
        by = sum(sum(per_cls.get(c, [])) for c in cls) if name != "hodge_general" else None  # one step
        rec = {"classes": cls, "ms_per_step": t, "share": t / step_phase}
        if by:
            rec.update({"algo_bytes_per_step": by, "gbs": by / (t * 1e-3) / 1e9, "frac": by / (t * 1e-3) / 1e9 / peak})
        func[name] = rec
    hf = [f for f in hodge_flops(pl, S, p, n) if f]
    fpk, fpk_src = fp64_peak()
    if hf and "hodge_general" in kernels:
        kernels["hodge_general"]["algo_flops"] = sum(hf) / len(hf)
        kernels["hodge_general"]["tflops"] = sum(hf) / len(hf) / (kernels["hodge_general"]["ms_per_launch"] * 1e-3) / 1e12
        wq = pl.qp_count() * (6 if pl.geom else 1) * 8
        hb = [b for c, b in lb if c == "hodge_general"]
        func["hodge_general"].update({"tflops": kernels["hodge_general"]["tflops"], "frac_fp64": kernels["hodge_general"]["tflops"] / fpk,
                                      "gbs": (sum(hb) / len(hb)) / (kernels["hodge_general"]["ms_per_launch"] * 1e-3) / 1e9,
                                      "weights_bytes": wq})
        func["hodge_general"]["frac"] = func["hodge_general"]["gbs"] / peak
    dom = max(func.items(), key=lambda kv: kv[1]["ms_per_step"])[0]
    # ncu DRAM bytes (dram__bytes_read + dram__bytes_write) of the dominant function per step, from the
    # committed full capture (profiles/traffic.json: per class, per launch)
    traffic = None
    tfile = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tfile):
        try:
            tj = json.load(open(tfile)).get(f"{args.config}_p{p}_n{n}", {})
            if all(c in tj for c in func[dom]["classes"]):
                traffic = sum(tj[c] * (prof[c][1] / K) for c in func[dom]["classes"])
        except Exception:
            traffic = None
    D = func[dom]
    t_step = ms / K * 1e-3
    roof = {"bound": "hbm", "kernel": dom, "achieved": D.get("gbs"), "peak": peak, "unit": "GB/s",
            "frac": D.get("frac"), "traffic": traffic, "peak_source": peak_src,
            "algo_bytes_per_step": D.get("algo_bytes_per_step"), "traffic_unit": "bytes per step (ncu)",
            "ms_per_step_in_kernel": D["ms_per_step"],
            "share_of_step": D["share"],
            "step_algo_bytes": step_bytes, "step_gbs": step_bytes / t_step / 1e9,
            "step_frac": step_bytes / t_step / 1e9 / peak,
            "bytes_per_dof_update": step_bytes / dofs,
            "useful_bytes_frac": 16.0 * dofs / t_step / 1e9 / peak,
            "functions": func,
            "note": "dominant = the kernel function (sweeps of every class / update / general Hodge) with the "
                    "largest wall time per step in the event-profiled pass (concurrent launches counted once); "
                    "achieved = its algorithmic bytes (DESIGN.md section 6) / that time; step_* = the unprofiled "
                    "timed pass against the step's algorithmic bytes; useful_bytes_frac = the algorithmic "
                    "minimum 16 B per DOF-update (read and write d and b once, SURVEY 8(d)) at the measured "
                    "step time, over the peak"}
    if dom == "hodge_general" and "tflops" in D:
        # the general Hodge is reported against the roof it is nearer to: fp64 arithmetic (scalar W at
        # p = 4: few W bytes per flop) or HBM (full W: 48 B of W per quadrature point);
        # the other view rides along
        alu_view = {"achieved": D["tflops"], "peak": fpk, "unit": "TFLOP/s", "frac": D["frac_fp64"],
                    "peak_source": fpk_src}
        if D["frac_fp64"] >= D["frac"]:
            roof.update({"bound": "alu", "achieved": D["tflops"], "peak": fpk, "unit": "TFLOP/s",
                         "frac": D["frac_fp64"], "peak_source": fpk_src,
                         "hbm_view": {"achieved": D["gbs"], "peak": peak, "unit": "GB/s", "frac": D["frac"]}})
        else:
            roof["alu_view"] = alu_view
        roof["algo_flops_per_launch"] = kernels["hodge_general"]["algo_flops"]

    # the structure-faithful three-axis schedule (every Kronecker factor swept) and the
    # fused-update schedule, timed the same way on the same state (second and third numbers)
    variants = {}
    if (pl.separable(S.MASS_EPS) and pl.separable(S.MASS_MU) and not getattr(args, "opts", 0)
            and not args.no_variants):
        for name, o in (("full_schedule", S.OPT_FULL_SCHEDULE), ("fused_update", S.OPT_FUSED)):
            pl.set_options(o)
            steps(0, W)
            torch.cuda.synchronize()
            vms, _ = timed(False)
            vms = max_over_ranks(vms, dist, dev)
            variants[name] = {"options": o, "ms_per_step": vms / K, "value": aggregate_value(dofs, K, vms, world),
                              "kernels_per_step": pl.kernels_per_step(),
                              "useful_bytes_frac": 16.0 * dofs / (vms / K * 1e-3) / 1e9 / peak}
        pl.set_options(0)
        # the (e,h)-state variant (sgm_step_eh, NEXT #3): two stored vectors, same DOF-updates
        for name, o in (("eh_state", 0), ("eh_state_fused", S.OPT_FUSED)):
            pl.set_options(o)
            e2, h2 = state[1].clone(), state[3].clone()
            pl.step_eh(e2, h2, dt, W, stream=stream)
            torch.cuda.synchronize()
            e0_, e1_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0_.record(stream)
            pl.step_eh(e2, h2, dt, K, stream=stream)
            e1_.record(stream)
            torch.cuda.synchronize()
            vms = max_over_ranks(e0_.elapsed_time(e1_), dist, dev)
            variants[name] = {"options": o, "ms_per_step": vms / K, "value": aggregate_value(dofs, K, vms, world),
                              "algo_bytes_per_dof_update": (8.0 if o else 12.0),
                              "useful_bytes_frac": 16.0 * dofs / (vms / K * 1e-3) / 1e9 / peak}
            del e2, h2
        pl.set_options(0)
    if (args.config == "c3" and not getattr(args, "opts", 0) and not args.no_variants):
        # on-the-fly DF in the general Hodge (SGM_OPT_OTF_GEOMETRY, NEXT #3): the two curved stars read
        # w_q / material (1 double per quadrature point) instead of the 6-entry weights
        n_qp = (n ** 3 if isinstance(n, int) else int(np.prod(n))) * (p + 1) ** 3
        w_full = 2 * 6 * 8.0 * n_qp / dofs
        pl.set_options(S.OPT_OTF_GEOMETRY)
        steps(0, W)
        torch.cuda.synchronize()
        vms, _ = timed(False)
        vms = max_over_ranks(vms, dist, dev)
        variants["otf_geometry"] = {"options": S.OPT_OTF_GEOMETRY, "ms_per_step": vms / K,
                                    "value": aggregate_value(dofs, K, vms, world),
                                    "w_bytes_per_dof_update": w_full / 6.0,
                                    "w_bytes_per_dof_update_stored": w_full}
        pl.set_options(0)
    env = {k: v for k, v in os.environ.items() if k.startswith("SGM_")}

    out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": W,
           "ms_per_step": ms / K, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
           "dtype": "f64", "data": "synthetic",
           "config": {"workload": desc, "p": p, "n_el": n, "dofs_per_step": dofs, "N_e": N_e, "N_h": N_h,
                      "parallelism": f"replicas x{world}" if world > 1 else "single GPU",
                      "l2": f"no flush: working set {(2 * N_e + 2 * N_h + max(N_e, N_h)) * 8 / 1e6:.0f} MB "
                            f"(state + workspace) vs 126 MB L2"},
           "roofline": roof, "kernels": kernels, "schedule_variants": variants,
           "schedule": {"mode": mode, "options": getattr(args, "opts", 0), "kernels_per_step": pl.kernels_per_step(),
                        "env_SGM": env, "dt": dt},
           "gpu_launches": pl.kernels_per_step() * K,
           "clocks": clk.summary()}

    # end to end through the public API, as a simulation uses it: the initial state is uploaded from
    # pinned host memory and the final state read back inside the timed region; every step uploads
    # its source amplitude s_k (the step's input) and reads back the step's monitor to the
    # host, the discrete Gauss-law residuals ||D~2 d||, ||D2 b||; the discrete energy
    # is read back once at the end.
    if not args.no_e2e:
        hs = [torch.empty(x.numel(), dtype=torch.float64, pin_memory=True) for x in state]
        for hx, x in zip(hs, state):
            hx.copy_(x)
        state_b = 8 * (2 * N_e + 2 * N_h)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        # (1) e2e through the C ABI with HOST buffers: one sgm_step_host call for the K steps -- the
        # pinned state (and source) host -> device, K steps, the state device -> host, synchronised
        jh = ja = None
        if jhat is not None:
            jh = torch.empty(N_e, dtype=torch.float64, pin_memory=True)
            jh.copy_(jhat)
            ja = torch.empty(K, dtype=torch.float64, pin_memory=True)
            ja.copy_(jamp[W:W + K])
        hs2 = [torch.empty(x.numel(), dtype=torch.float64, pin_memory=True) for x in hs]  # (empty_like: pageable)
        for a_, b_ in zip(hs2, hs):
            a_.copy_(b_)
        pl.step_host(*hs2, dt, K, j_hat=jh, j_amp=ja, stream=stream)  # allocates the mirrors (untimed)
        for a_, b_ in zip(hs2, hs):
            a_.copy_(b_)
        torch.cuda.synchronize()
        e0.record(stream)
        pl.step_host(*hs2, dt, K, j_hat=jh, j_amp=ja, stream=stream)
        e1.record(stream)
        torch.cuda.synchronize()
        ems0 = max_over_ranks(e0.elapsed_time(e1), dist, dev)
        # sgm_step_host uploads d, b, h (e is recomputed from d before any use, sgm.h) and j^, s_k
        h2d = 8 * (N_e + 2 * N_h) + (8 * N_e + 8 * K if jh is not None else 0)
        out["e2e"] = {"value": aggregate_value(dofs, K, ems0, world), "unit": UNIT,
                      "h2d_bytes_per_step": h2d / K, "d2h_bytes_per_step": state_b / K, "steps": K,
                      "note": "C-ABI sgm_step_host on pinned HOST buffers: d, b, h (and j^, s_k) host->device, "
                              "K steps, d, e, b, h device->host, all inside the CUDA-event region on the stream"}
        del hs2
        # (2) a simulation loop through the public API: state up once, per step s_k up, sgm_step,
        # the Gauss-law residuals down, energy and the state down at the end
        amp_h = torch.ones(K, dtype=torch.float64, pin_memory=True)
        amp_d = torch.empty(K, dtype=torch.float64, device=dev)
        en_d = torch.zeros(2, dtype=torch.float64, device=dev)
        en_h = torch.zeros(2 * K + 1, dtype=torch.float64, pin_memory=True)
        dv = [torch.empty_like(x) for x in state]
        torch.cuda.synchronize()
        e0.record(stream)
        for i in (0, 2, 3):
            dv[i].copy_(hs[i], non_blocking=True)
        for k in range(K):
            amp_d[k:k + 1].copy_(amp_h[k:k + 1], non_blocking=True)
            pl.step(*dv, dt, 1, j_hat=jhat, j_amp=amp_d[k:k + 1] if jhat is not None else None, stream=stream)
            pl.gauss(dv[0], dv[2], en_d, stream=stream)
            en_h[2 * k:2 * k + 2].copy_(en_d, non_blocking=True)
        pl.energy(*dv, en_d, stream=stream)
        en_h[2 * K:2 * K + 1].copy_(en_d[:1], non_blocking=True)
        for x, hx in zip(dv, hs):
            hx.copy_(x, non_blocking=True)
        e1.record(stream)
        torch.cuda.synchronize()
        ems = max_over_ranks(e0.elapsed_time(e1), dist, dev)
        in_b = 8 * (N_e + 2 * N_h)
        out["e2e_loop"] = {"value": aggregate_value(dofs, K, ems, world), "unit": UNIT,
                           "h2d_bytes_per_step": in_b / K + 8, "d2h_bytes_per_step": state_b / K + 16 + 8 / K,
                           "steps": K, "gauss_last": [float(en_h[2 * K - 2]), float(en_h[2 * K - 1])],
                           "energy_end": float(en_h[2 * K]),
                           "note": "public API loop: initial state (d, b, h; e is recomputed from d by the first "
                                   "half-step) H2D and final state D2H, pinned, inside the timed region; per step "
                                   "s_k H2D, sgm_step, sgm_gauss, residuals D2H; energy D2H at the end"}
        # the pessimistic variant: the whole state crosses PCIe both ways every step (sgm_step_host)
        ke = min(K, 10)
        pl.step_host(*hs, dt, 1, stream=stream)
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(ke):
            pl.step_host(*hs, dt, 1, stream=stream)
        e1.record(stream)
        torch.cuda.synchronize()
        ems2 = max_over_ranks(e0.elapsed_time(e1), dist, dev)
        out["e2e_state_roundtrip"] = {"value": aggregate_value(dofs, ke, ems2, world), "unit": UNIT,
                                      "h2d_bytes_per_step": state_b, "d2h_bytes_per_step": state_b, "steps": ke,
                                      "note": "sgm_step_host: pinned d,e,b,h -> device, 1 step, -> host, every step"}

    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            out["cpu_baseline"] = cpu_baseline(args)
        except Exception as ex:  # the baseline is informational
            out["cpu_baseline"] = {"value": None, "error": str(ex)}
    if rank == 0:
        print(json.dumps(out))
    if dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
