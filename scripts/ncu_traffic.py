#!/usr/bin/env python
"""From an `ncu --set full` raw CSV of one step's 8 launches (update, z, y, x for the eps half, then
the mu half), write per-class DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum, bytes per
launch) into profiles/traffic.json under the given workload key, and print a markdown table.
    python scripts/ncu_traffic.py RAW_CSV KEY"""
import csv
import json
import os
import sys

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
raw, key = sys.argv[1], sys.argv[2]
rows = list(csv.reader(open(raw)))
hdr, units, data = rows[0], rows[1], rows[2:]

# one step from the first Ampere update: update, eps passes, update, mu passes.  The eps half has
# 3 sweep launches; the mu half 3, or 2 when its z and y sweeps share a launch (reduced schedule).
names = [d[hdr.index("Kernel Name")] for d in data]
start = next(i for i, nm in enumerate(names) if "update_kernel<1" in nm)
nxt = next(i for i in range(start + 1, len(names)) if "update_kernel<2" in names[i])
end = next((i for i in range(nxt + 1, len(names)) if "update_kernel" in names[i]), len(names))
n_mu = end - nxt - 1
CLASSES = ["update", "eps_z", "eps_y", "eps_x", "update"] + (["mu_z", "mu_x"] if n_mu == 2 else ["mu_z", "mu_y", "mu_x"])
data = data[start:end]


def col(name, d):
    i = hdr.index(name)
    return float(d[i]) * UNIT.get(units[i], 1)


traffic, table = {}, []
for cls, d in zip(CLASSES, data):
    rd, wr = col("dram__bytes_read.sum", d), col("dram__bytes_write.sum", d)
    t = col("gpu__time_duration.sum", d) if units[hdr.index("gpu__time_duration.sum")] != "us" else float(
        d[hdr.index("gpu__time_duration.sum")]) * 1e-6
    traffic.setdefault(cls, []).append(rd + wr)
    table.append((cls, d[hdr.index("Kernel Name")][:60], rd / 1e6, wr / 1e6,
                  float(d[hdr.index("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed")]),
                  float(d[hdr.index("sm__inst_executed.avg.per_cycle_active")]),
                  float(d[hdr.index("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active")]),
                  float(d[hdr.index("gpu__time_duration.sum")])))
path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "traffic.json")
allt = json.load(open(path)) if os.path.exists(path) else {}
allt[key] = {k: sum(v) / len(v) for k, v in traffic.items()}
json.dump(allt, open(path, "w"), indent=1)
print("| class | kernel | DRAM read MB | DRAM write MB | DRAM % peak | IPC | fp64 pipe % | time (us, ncu) |")
print("|---|---|---|---|---|---|---|---|")
for r in table:
    print("| %s | `%s` | %.1f | %.1f | %.1f | %.2f | %.1f | %.1f |" % r)
