"""Per-CUDA-source-line instruction counts and stall samples from an ncu report's cuda,sass view
(`ncu -i X.ncu-rep --page source --csv --print-source cuda,sass`)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
f = None
ln = None
hdr = None
ex = collections.Counter()
st = collections.Counter()
ops = collections.defaultdict(collections.Counter)
srcline = {}
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8:
        continue
    if r[0]:
        ln = (f, int(r[0]))
        srcline[ln] = r[1]
        continue
    try:
        e = float(r[hdr.index("Instructions Executed")] or 0)
        s = float(r[4] or 0)
    except ValueError:
        continue
    ex[ln] += e
    st[ln] += s
    op = r[3].split()
    op = (op[1] if op and op[0].startswith("@") else (op[0] if op else "?")).split(".")[0]
    ops[ln][op] += e
T = sum(ex.values())
S = sum(st.values())
print(f"total {T:.0f} warp-instructions, {S:.0f} stall samples")
for ln, e in sorted(ex.items(), key=lambda kv: -kv[1])[:top]:
    o = " ".join(f"{k}:{v/1e3:.0f}k" for k, v in ops[ln].most_common(5))
    print(f"{ln[0]}:{ln[1]:4d} {100*e/T:5.1f}% inst {100*st[ln]/S:5.1f}% stall | {srcline.get(ln,'').strip()[:60]:60s} | {o}")
