#!/usr/bin/env python
"""Per-CUDA-source-line warp-stall samples of one kernel in an ncu report.

    python scripts/ncu_lines.py REPORT.ncu-rep KERNEL_REGEX [launch_index] [top]
Runs `ncu -i REPORT --page source --csv --print-source cuda,sass` for one launch and sums the
stall samples of the SASS under each CUDA line (needs -lineinfo and --import-source on)."""
import csv
import io
import subprocess
import sys


def main(rep, kre, idx=0, top=30):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                          "-k", "regex:" + kre, "--launch-skip", str(idx), "--launch-count", "1"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = None
    agg = {}
    cur = None
    fname = ""
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Function Name":
            print("#", r[1][:120])
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None:
            continue
        if r[0]:
            cur = (fname, int(r[0]), r[1].strip())
            continue
        if cur is None or r[2] in ("...", "-"):
            continue
        d = agg.setdefault(cur, {"samples": 0, "inst": 0, "stalls": {}})
        try:
            d["samples"] += int(r[4])
            d["inst"] += int(r[7])
        except ValueError:
            continue
        for j, h in enumerate(hdr):
            if h.startswith("stall_") and "Not Issued" not in h:
                try:
                    v = int(r[j])
                except ValueError:
                    continue
                if v:
                    d["stalls"][h[6:]] = d["stalls"].get(h[6:], 0) + v
    tot = sum(d["samples"] for d in agg.values()) or 1
    print(f"total samples {tot}")
    for k, d in sorted(agg.items(), key=lambda kv: -kv[1]["samples"])[:top]:
        st = ", ".join(f"{n}={v}" for n, v in sorted(d["stalls"].items(), key=lambda x: -x[1])[:3])
        print(f"{100 * d['samples'] / tot:5.1f}% {d['samples']:6d} inst={d['inst']:8d} {k[0]}:{k[1]:4d} {k[2][:70]:70s} {st}")


if __name__ == "__main__":
    a = sys.argv
    main(a[1], a[2], int(a[3]) if len(a) > 3 else 0, int(a[4]) if len(a) > 4 else 30)
