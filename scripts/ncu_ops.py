#!/usr/bin/env python
"""Dynamic SASS opcode mix of one launch in an ncu report (per N elements if given).
    python scripts/ncu_ops.py REPORT KERNEL_REGEX LAUNCH_INDEX [elements]"""
import collections
import csv
import io
import re
import subprocess
import sys

rep, kre, idx = sys.argv[1], sys.argv[2], int(sys.argv[3])
elems = float(sys.argv[4]) if len(sys.argv) > 4 else None
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", "regex:" + kre,
                      "--launch-skip", str(idx), "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = None
cnt, samp = collections.Counter(), collections.Counter()
seen = set()
for r in rows:
    if r and r[0] == "Address":
        hdr = r
        continue
    if hdr is None or len(r) < 6 or not r[0].startswith("0x") or r[0] in seen:
        continue
    seen.add(r[0])
    op = re.sub(r"^@!?U?P\w+\s+", "", r[1].strip()).split()[0]
    base = op.split(".")[0]
    if base in ("LDS", "STS", "LDG", "STG", "LDGSTS"):
        base = op
    cnt[base] += int(r[hdr.index("Instructions Executed")] or 0)
    samp[base] += int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
tot = sum(cnt.values())
st = sum(samp.values()) or 1
print(f"total warp-instructions {tot}" + (f"  per 32 elements {32 * tot / elems:.1f}" if elems else ""))
for op, c in cnt.most_common(30):
    per = f"{32 * c / elems:6.2f}" if elems else ""
    print(f"{op:14s} {c:10d} {per}  stall-samples {100 * samp[op] / st:5.1f}%")
