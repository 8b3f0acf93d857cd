#!/usr/bin/env python
"""Copy one scripts/gpu_full_r2.sh run (TAG) from gpurun_out/ into profiles/ (r2_* files) and write
profiles/r2_summary.md.      python scripts/make_summary_r2.py TAG"""
import csv
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(ROOT, "gpurun_out")
PR = os.path.join(ROOT, "profiles")
sys.path.insert(0, os.path.join(ROOT, "scripts"))
from make_summary import launch_shares  # noqa: E402

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3,
        "ns": 1e-3, "us": 1.0, "ms": 1e3}


def ncu_rows(path):
    rows = list(csv.reader(open(path)))
    hdr, units, data = rows[0], rows[1], rows[2:]

    def get(d, name):
        if name not in hdr:
            return None
        i = hdr.index(name)
        try:
            return float(d[i].replace(",", "")) * UNIT.get(units[i], 1)
        except ValueError:
            return None
    out = []
    for d in data:
        out.append({"kernel": d[hdr.index("Kernel Name")].split("(")[0][-60:],
                    "us": get(d, "gpu__time_duration.sum"),
                    "dram_mb": ((get(d, "dram__bytes_read.sum") or 0) + (get(d, "dram__bytes_write.sum") or 0)) / 1e6,
                    "ipc": get(d, "sm__inst_executed.avg.per_cycle_active"),
                    "fp64": get(d, "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
                    "conf": get(d, "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"),
                    "warps": get(d, "sm__warps_active.avg.pct_of_peak_sustained_active")})
    return out


def main(tag, htag=None):
    cp = lambda src, dst: shutil.copy(os.path.join(G, src), os.path.join(PR, dst))  # noqa: E731
    b = json.load(open(os.path.join(G, f"bench_{tag}.json")))
    ref = json.load(open(os.path.join(G, f"bench_ref_{tag}.json")))
    sweep = [json.loads(l) for l in open(os.path.join(G, f"bench_sweep_{tag}.jsonl")) if l.strip()]
    cp(f"bench_{tag}.json", "r2_bench.json")
    cp(f"bench_ref_{tag}.json", "r2_bench_reference.json")
    if htag:
        # general-Hodge workloads (C4, C3), the brick kernel's ncu captures and the test logs from a later
        # call (scripts/gpu_s5e.sh) on the final library
        sweep = [d for d in sweep if d["roofline"]["kernel"] != "hodge_general"]
        sweep += [json.loads(l) for l in open(os.path.join(G, f"bench_hodge_{htag}.jsonl")) if l.strip()]
        with open(os.path.join(PR, "r2_bench_sweep.jsonl"), "w") as fh:
            for d in sweep:
                fh.write(json.dumps(d) + "\n")
    else:
        cp(f"bench_sweep_{tag}.jsonl", "r2_bench_sweep.jsonl")
    cp(f"launches_{tag}.csv", "r2_ncu_launches.csv")
    cp(f"full_{tag}_raw.csv", "r2_ncu_full_raw.csv")
    for c in ("c3", "c4"):
        if os.path.exists(os.path.join(G, f"hodge_{c}_{htag or tag}_raw.csv")):
            cp(f"hodge_{c}_{htag or tag}_raw.csv", f"r2_ncu_hodge_{c}_raw.csv")
    if os.path.exists(os.path.join(G, f"c5_sweep_{tag}.jsonl")):
        cp(f"c5_sweep_{tag}.jsonl", "r2_c5_sweep.jsonl")
    table = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "ncu_traffic.py"),
                            os.path.join(G, f"full_{tag}_raw.csv"), "c5_p3_n128"],
                           capture_output=True, text=True).stdout
    ser, shares = launch_shares(os.path.join(G, f"launches_{tag}.csv"))
    pyt = open(os.path.join(G, f"pytest_gpu_{htag or tag}.log")).read().strip().splitlines()[-1]
    smoke = open(os.path.join(G, f"smoke_{htag or tag}.log")).read().strip().splitlines()[-1]
    r = b["roofline"]
    L = ["# Round 2 profile summary (B200, sm_100a)\n",
         f"From one `gpurun` call (`TAG={tag} bash scripts/gpu_full_r2.sh`), summarised by "
         f"`python scripts/make_summary_r2.py {tag}`" + (f"; the general-Hodge workloads (C4, C3 lines, brick-kernel "
         f"ncu captures) and the test / smoke lines below from a later call on the final library "
         f"(`TAG={htag} bash scripts/gpu_s5e.sh`)" if htag else "") + ". Round-1 files (`r1_*`) are kept for comparison.\n",
         f"Same call: `pytest -m \"gpu and not slow\"` → {pyt}; `smoke()` → {smoke}. The full-size parity "
         "(`-m \"gpu and slow\"`, C3 200 and C4 100 steps as configured, C5 at 100 steps) is in "
         "`r2_parity_fullsize.md`; the measured fp64 peak in `r2_fp64_peak.json`.\n",
         "## Headline: C5 p=3 128³ (bench default, unprofiled, CUDA events)\n"]
    c = b["clocks"]
    L.append(f"* **{b['value']:.3e} DOF-updates/s**, {1e3 * b['ms_per_step']:.1f} µs per step, clocks "
             f"{c['sm_mhz']:.0f}/{c['sm_max_mhz']} MHz, throttle reasons {c['reasons'] or 'none'}, "
             f"{b['schedule']['kernels_per_step']} kernels per step, options {b['schedule']['options']}, SGM_* env {b['schedule']['env_SGM'] or 'none'}")
    L.append(f"* step: {r['step_algo_bytes'] / 1e6:.0f} MB algorithmic ({r['bytes_per_dof_update']:.0f} B per DOF-update) → "
             f"{r['step_gbs']:.0f} GB/s = **{r['step_frac']:.2f}** of the measured {r['peak']} GB/s; useful-bytes "
             f"fraction (16 B per DOF-update) **{r['useful_bytes_frac']:.2f}**")
    L.append(f"* dominant kernel function `{r['kernel']}` ({100 * r['share_of_step']:.0f} % of the step's kernel time): "
             f"{r['achieved']:.0f} GB/s = **{r['frac']:.2f}** of peak"
             + (f"; ncu DRAM {r['traffic'] / 1e6:.0f} MB per step vs {r['algo_bytes_per_step'] / 1e6:.0f} MB algorithmic"
                if r.get("traffic") else ""))
    L.append("\n| function | classes | ms per step | algorithmic MB per step | GB/s | frac of peak |")
    L.append("|---|---|---|---|---|---|")
    for k, f in r["functions"].items():
        L.append(f"| {k} | {', '.join(f['classes'])} | {f['ms_per_step']:.4f} | "
                 f"{(f.get('algo_bytes_per_step') or 0) / 1e6:.0f} | {f.get('gbs', 0):.0f} | {f.get('frac', 0):.2f} |")
    L.append("\nSchedule variants on the same state (`schedule_variants`):\n")
    L.append("| variant | ms per step | DOF-updates/s | useful-bytes frac |")
    L.append("|---|---|---|---|")
    L.append(f"| default (reduced, concurrent pairs) | {b['ms_per_step']:.4f} | {b['value']:.3e} | {r['useful_bytes_frac']:.2f} |")
    for k, v in b.get("schedule_variants", {}).items():
        L.append(f"| {k} | {v['ms_per_step']:.4f} | {v['value']:.3e} | {v['useful_bytes_frac']:.2f} |")
    L.append(f"\n* e2e (C ABI on pinned host buffers, `sgm_step_host` over the {b['e2e']['steps']} steps): "
             f"{b['e2e']['value']:.3e} DOF-updates/s; simulation loop (`e2e_loop`): {b['e2e_loop']['value']:.3e}; "
             f"full state round trip every step: {b['e2e_state_roundtrip']['value']:.3e}")
    L.append(f"* CPU oracle on the box's {b['cpu_baseline']['cores']} host threads: {b['cpu_baseline']['value']:.3e} "
             f"DOF-updates/s (reference arm: {ref.get('value', float('nan')):.3e})\n")
    L.append("## Other workloads (`--steps 20 --warmup 5`)\n")
    L.append("| workload | DOF-updates/s | ms/step | dominant (frac of its peak) | step HBM frac | CPU oracle DOF-updates/s |")
    L.append("|---|---|---|---|---|---|")
    for d in sweep:
        rr = dict(d["roofline"])
        hv = rr.get("hbm_view")
        if hv and hv["frac"] > rr["frac"]:  # lines written before bench.py picked the nearer roof itself
            rr.update({"achieved": hv["achieved"], "unit": hv["unit"], "frac": hv["frac"]})
        cb = d.get("cpu_baseline") or {}
        L.append(f"| {d['config']['workload']} | {d['value']:.3g} | {d['ms_per_step']:.3f} | {rr['kernel']} "
                 f"{rr['achieved']:.3g} {rr['unit']} ({rr['frac']:.2f}) | {rr.get('step_frac', 0):.2f} | "
                 f"{cb.get('value') or float('nan'):.3g} |")
    for d in sweep:
        for k, v in d.get("schedule_variants", {}).items():
            extra = (f", W bytes per DOF-update {v['w_bytes_per_dof_update_stored']:.0f} -> "
                     f"{v['w_bytes_per_dof_update']:.0f}" if "w_bytes_per_dof_update" in v else "")
            L.append(f"* {d['config']['workload'].split(' ')[0]} variant `{k}` (options {v['options']}): "
                     f"{v['ms_per_step']:.3f} ms per step (default {d['ms_per_step']:.3f}){extra}")
    c5p = os.path.join(PR, "r2_c5_sweep.jsonl")
    if os.path.exists(c5p):
        L.append("\n## configs[4]: K1 wedge solve and full step over p and n (`scripts/c5_sweep.py`)\n")
        L.append("| p | n_el | K1 solve µs | solve GB/s (frac) | step µs | DOF-updates/s | step GB/s (frac) |")
        L.append("|---|---|---|---|---|---|---|")
        for l in open(c5p):
            d = json.loads(l)
            k, s_ = d["kron_solve"], d["step"]
            L.append(f"| {d['p']} | {d['n_el']} | {k['us']:.1f} | {k['gbs']:.0f} ({k['frac']:.2f}) | {s_['us']:.1f} | "
                     f"{s_['dof_updates_per_s']:.3g} | {s_['gbs']:.0f} ({s_['frac']:.2f}) |")
    L.append("\n## ncu, one step of C5 p=3 128³ (serialised replay: compare shares, not absolutes)\n")
    L.append(table.strip() + "\n")
    L.append(f"Launch-list shares (last 3 steps of `r2_ncu_launches.csv`, serialised step {ser:.0f} µs): " +
             ", ".join(f"{n} {s:.0f} %" for n, s in shares) + ".\n")
    for cc in ("c3", "c4"):
        pth = os.path.join(PR, f"r2_ncu_hodge_{cc}_raw.csv")
        if os.path.exists(pth):
            L.append(f"### General Hodge, {cc.upper()} (`r2_ncu_hodge_{cc}_raw.csv`)\n")
            L.append("| kernel | µs | DRAM MB | IPC | fp64 pipe % | smem bank conflicts | warps active % |")
            L.append("|---|---|---|---|---|---|---|")
            for x in ncu_rows(pth):
                L.append(f"| `{x['kernel']}` | {x['us'] or 0:.1f} | {x['dram_mb']:.0f} | {x['ipc'] or 0:.2f} | "
                         f"{x['fp64'] or 0:.1f} | {x['conf'] or 0:.3g} | {x['warps'] or 0:.1f} |")
            L.append("")
    open(os.path.join(PR, "r2_summary.md"), "w").write("\n".join(L) + "\n")
    print("\n".join(L))


if __name__ == "__main__":
    main(*sys.argv[1:3])
