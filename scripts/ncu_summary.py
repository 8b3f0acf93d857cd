#!/usr/bin/env python
"""Summarise an `ncu --page raw --csv` export: one block per profiled launch with the metrics
that matter for the line sweeps (duration, DRAM bytes and throughput, occupancy, IPC, fp64 pipe,
registers, stall reasons).  Usage: python scripts/ncu_summary.py gpurun_out/full_X_raw.csv"""
import csv
import sys

KEYS = [
    ("Kernel Name", "kernel"),
    ("Grid Size", "grid"),
    ("Block Size", "block"),
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram_rd"),
    ("dram__bytes_write.sum", "dram_wr"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_%peak"),
    ("lts__t_bytes.sum", "l2_bytes"),
    ("launch__registers_per_thread", "regs"),
    ("launch__occupancy_limit_registers", "occ_lim_regs"),
    ("launch__occupancy_limit_shared_mem", "occ_lim_smem"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_active%"),
    ("sm__inst_executed.avg.per_cycle_active", "ipc"),
    ("smsp__inst_executed.sum", "inst"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64_pipe%"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem_conflicts"),
]


def main(path):
    rows = list(csv.reader(open(path)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    pre, suf = "smsp__average_warps_issue_stalled_", "_per_issue_active.ratio"
    stall_cols = [i for i, h in enumerate(hdr) if h.startswith(pre) and h.endswith(suf)]
    for d in data:
        print("-" * 80)
        for k, short in KEYS:
            if k in hdr:
                i = hdr.index(k)
                print(f"  {short:16s} {d[i]} {units[i]}")
        # top stall reasons (warp-cycles per issued instruction)
        st = []
        for i in stall_cols:
            try:
                st.append((float(d[i]), hdr[i][len(pre):-len(suf)]))
            except ValueError:
                pass
        st.sort(reverse=True)
        print("  top stalls:", ", ".join(f"{n}={v:.2f}" for v, n in st[:6]))


if __name__ == "__main__":
    main(sys.argv[1])
