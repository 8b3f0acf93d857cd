#!/usr/bin/env python
"""Copy one gpu_full.sh run (TAG) from gpurun_out/ into profiles/ and write profiles/r1_summary.md.

    python scripts/make_summary.py TAG
Reads bench_TAG.json, bench_ref_TAG.json, bench_sweep_TAG.jsonl, launches_TAG.csv, full_TAG_raw.csv,
pytest_gpu_TAG.log and smoke_TAG.log; updates profiles/traffic.json (scripts/ncu_traffic.py)."""
import collections
import csv
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(ROOT, "gpurun_out")
PR = os.path.join(ROOT, "profiles")


def launch_shares(path):
    rows = list(csv.reader(open(path)))
    i = next(k for k, r in enumerate(rows) if "Kernel Name" in r)
    hdr, data = rows[i], rows[i + 1:]
    kn, mv, mn = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
    ts = [(r[kn], float(r[mv].replace(",", ""))) for r in data if r[mn] == "gpu__time_duration.sum"]
    starts = [k for k, (n, _) in enumerate(ts) if "update_kernel<1" in n]
    last = ts[starts[-3]:]
    agg = collections.OrderedDict()
    for n, t in last:
        if "update_kernel<1" in n:
            c = "Ampère update"
        elif "update_kernel<2" in n:
            c = "Faraday update"
        elif "sweep_kernel" in n:
            c = "sweeps"
        else:
            c = n.split("(")[0][-40:]
        agg[c] = agg.get(c, 0.0) + t
    tot = sum(agg.values())
    return tot / 3 / 1000.0, [(c, 100 * t / tot) for c, t in agg.items()]


def main(tag):
    b = json.load(open(os.path.join(G, f"bench_{tag}.json")))
    ref = json.load(open(os.path.join(G, f"bench_ref_{tag}.json")))
    sweep = [json.loads(l) for l in open(os.path.join(G, f"bench_sweep_{tag}.jsonl"))]
    shutil.copy(os.path.join(G, f"bench_{tag}.json"), os.path.join(PR, "r1_bench.json"))
    shutil.copy(os.path.join(G, f"bench_ref_{tag}.json"), os.path.join(PR, "r1_bench_reference.json"))
    shutil.copy(os.path.join(G, f"bench_sweep_{tag}.jsonl"), os.path.join(PR, "r1_bench_sweep.jsonl"))
    shutil.copy(os.path.join(G, f"launches_{tag}.csv"), os.path.join(PR, "r1_ncu_launches.csv"))
    shutil.copy(os.path.join(G, f"full_{tag}_raw.csv"), os.path.join(PR, "r1_ncu_full_raw.csv"))
    table = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "ncu_traffic.py"),
                            os.path.join(G, f"full_{tag}_raw.csv"), "c5_p3_n128"],
                           capture_output=True, text=True, check=True).stdout
    ser, shares = launch_shares(os.path.join(G, f"launches_{tag}.csv"))
    pyt = open(os.path.join(G, f"pytest_gpu_{tag}.log")).read().strip().splitlines()[-1]
    smoke = open(os.path.join(G, f"smoke_{tag}.log")).read().strip().splitlines()[-1]
    r = b["roofline"]
    L = []
    L.append("# Round 1 profile summary (B200, sm_100a)\n")
    L.append(f"Everything here comes from one `gpurun` call (`TAG={tag} bash scripts/gpu_full.sh`), summarised by "
             f"`python scripts/make_summary.py {tag}`. Earlier round-1 evidence is in git history.\n")
    L.append("Files:")
    L.append("* `r1_bench.json` — `python bench.py` (C5 p=3 128³, K=100, W=10, CUDA events, NVML clocks during the timed region)")
    L.append("* `r1_bench_reference.json` — `python bench.py --impl reference --steps 3 --warmup 1` (the CPU oracle, tier B)")
    L.append("* `r1_bench_sweep.jsonl` — other workloads (`--p 2 --n 160`, `--p 4 --n 128`, `--p 3 --n 64`, `--config c4`, `--config c3`)")
    L.append("* `r1_ncu_launches.csv` — `ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e`")
    L.append("* `r1_ncu_full_raw.csv` — `ncu --set full --clock-control none --import-source on -k \"regex:sweep_kernel|update_kernel\" --launch-skip 26 --launch-count 14` (two steps)")
    L.append("* `r1_ncu_hodge_brick_c4_raw.csv`, `r1_ncu_hodge_brick_c3_raw.csv` — `TAG=... KREGEX=hodge_brick ARGS=\"--config c4|c3 ...\" bash scripts/ncu_one.sh` (separate call): the general-Hodge brick kernel (C4 ε-Hodge 1.63 ms, IPC 1.25, fp64 pipe 17 %, 0.94 GB DRAM; C3 0.155 ms, IPC 0.98, fp64 pipe 10 %)")
    L.append("* `traffic.json` — per-class DRAM bytes per launch from the full capture (`scripts/ncu_traffic.py`, read by bench.py)")
    L.append("* `r1_cpu_oracle.jsonl` — `scripts/oracle_timing.py` (separate call): the CPU oracle per step for every config")
    L.append("* `r1_scheme_compare.md` — scheme 1 (mass-matrix Hodge stars) against scheme 2 on this GPU (separate calls)\n")
    L.append(f"Same call: `pytest -m gpu` → {pyt}; `smoke()` → {smoke}\n")
    L.append("## Headline (unprofiled, live)\n")
    c = b["clocks"]
    L.append(f"* **{b['value']:.3e} DOF-updates/s**, {1e3 * b['ms_per_step']:.1f} µs per step "
             f"({b['config']['dofs_per_step'] / 1e6:.2f} M DOF-updates per step), clocks {c['sm_mhz']:.0f}/{c['sm_max_mhz']} MHz, "
             f"throttle reasons {c['reasons'] or 'none'}")
    L.append(f"* whole step: {r['step_algo_bytes'] / 1e6:.0f} MB algorithmic → {r['step_gbs']:.0f} GB/s = "
             f"**{r['step_frac']:.2f} of the measured {r['peak']} GB/s**")
    L.append(f"* dominant kernel (largest share of the event-profiled pass): `{r['kernel']}` {r['achieved']:.0f} GB/s = "
             f"**{r['frac']:.2f}** of measured peak; ncu DRAM traffic {r['traffic'] / 1e6 if r['traffic'] else float('nan'):.0f} MB per launch "
             f"vs {r['algo_bytes_per_launch'] / 1e6:.0f} MB algorithmic")
    L.append(f"* e2e through the public API (state H2D once, per step s_k H2D + sgm_step + Gauss residuals D2H, "
             f"final state D2H): {b['e2e']['value']:.3e} DOF-updates/s")
    L.append(f"* CPU oracle on the box's {b['cpu_baseline']['cores']} host threads: {b['cpu_baseline']['value']:.3e} "
             f"DOF-updates/s (reference arm: {ref['value']:.3e})\n")
    L.append("## Other workloads (same binary, `--steps 20 --warmup 5`)\n")
    L.append("| workload | DOF-updates/s | ms/step | dominant kernel (frac of its peak) | step HBM frac |")
    L.append("|---|---|---|---|---|")
    for d in sweep:
        rr = d["roofline"]
        L.append(f"| {d['config']['workload']} | {d['value']:.3g} | {d['ms_per_step']:.3f} | {rr['kernel']} "
                 f"{rr['achieved']:.3g} {rr['unit']} ({rr['frac']:.2f}) | {rr.get('step_frac', 0):.2f} |")
    c5 = os.path.join(G, f"c5_sweep_{tag}.jsonl")
    if os.path.exists(c5):
        shutil.copy(c5, os.path.join(PR, "r1_c5_sweep.jsonl"))
    c5p = os.path.join(PR, "r1_c5_sweep.jsonl")
    if os.path.exists(c5p):
        L.append("\n### configs[4]: Kronecker wedge solve and full step over p and n (`scripts/c5_sweep.py`, `r1_c5_sweep.jsonl`)\n")
        L.append("K1 solve = `sgm_kron_solve` (three sweeps; 48 B/element algorithmic, L2 flushed before each rep); "
                 "step = `sgm_step` graph replay. Fractions of the measured HBM peak.\n")
        L.append("| p | n_el | K1 solve µs | solve GB/s (frac) | step µs | DOF-updates/s | step GB/s (frac) |")
        L.append("|---|---|---|---|---|---|---|")
        for l in open(c5p):
            d = json.loads(l)
            k, s_ = d["kron_solve"], d["step"]
            L.append(f"| {d['p']} | {d['n_el']} | {k['us']:.1f} | {k['gbs']:.0f} ({k['frac']:.2f}) | {s_['us']:.1f} | "
                     f"{s_['dof_updates_per_s']:.3g} | {s_['gbs']:.0f} ({s_['frac']:.2f}) |")
        L.append("\nAt 32³ and 64³ the working set sits in L2 and the kernels are launch/latency bound; at 160³ with "
                 "p ≥ 3 the strided sweeps have only two producer warps (14 consumer segments fill the 16-warp CTA) "
                 "and p = 4 no longer fits two lines per thread in shared memory.")
    co = os.path.join(PR, "r1_cpu_oracle.jsonl")
    if os.path.exists(co):
        L.append("\n### CPU oracle per step on the GPU box's host (`scripts/oracle_timing.py`, `r1_cpu_oracle.jsonl`)\n")
        L.append("The oracle as it stands (setup excluded, median of >= 3 steps after a warm-up); a reported "
                 "baseline, not the target. Tier A = assembled matrices + SuperLU, tier B = Kronecker.\n")
        L.append("| config | tier | s/step | DOF-updates/s | BLAS threads / cores |")
        L.append("|---|---|---|---|---|")
        for l in open(co):
            d = json.loads(l)
            L.append(f"| {d['config']} | {d['tier']} | {d['s_per_step']:.3g} | {d['dof_updates_per_s']:.3g} | "
                     f"{d['blas_threads']}/{d['cores']} |")
    L.append("\nC4/C3 report the general Hodge against the fp64 peak (`bound: alu`, 37.2 TFLOP/s, DESIGN.md §6); its "
             "HBM view is in each line's `roofline.hbm_view`.\n")
    L.append("## Per-kernel ncu, one step of C5 p=3 128³ (serialised replay: compare shares, not absolutes)\n")
    L.append(table.strip() + "\n")
    L.append(f"Launch-list shares (last 3 steps of `r1_ncu_launches.csv`, serialised step {ser:.0f} µs): " +
             ", ".join(f"{n} {s:.0f} %" for n, s in shares) + ". ncu serialises every launch, so the two "
             "concurrent sweep pairs per step (each side sized for its 1/3 or 2/3 share of the SMs) run one "
             "after the other there: the sweeps' share is inflated against the live step "
             f"({1e3 * b['ms_per_step']:.0f} µs, where the event-profiled pass gives the updates "
             f"{100 * b['kernels']['update']['ms_per_launch'] * b['kernels']['update']['launches'] / b['steps'] / b['ms_per_step']:.0f} %).\n")
    L.append("## Reading\n")
    L.append("* The **update** kernels stream ≈135 MB of DRAM per launch (156 MB algorithmic; ncu's replay flushes L2, "
             "so live L2 reuse is not visible here) and are memory-latency bound; a torch elementwise kernel with the "
             "same bytes takes 30 µs on this GPU (`scripts/micro_stream.py`).")
    L.append("* The **sweeps** read their algorithmic input bytes from DRAM and their writes stay in L2 for the next "
             "kernel; DRAM is 7–21 % busy: they are bound by the SPIKE consumers' instruction issue and per-tile "
             "latency (IPC 1.2–1.4, fp64 pipe ≈25 %). The concurrent pairs (ε y ∥ ε x, μ z+y ∥ μ x) each run on "
             "their share of the SMs.")
    open(os.path.join(PR, "r1_summary.md"), "w").write("\n".join(L) + "\n")
    print("\n".join(L))


if __name__ == "__main__":
    main(sys.argv[1])
