"""Timeline of one sweep launch (tuning build only: SGM_BUILD_TUNING=1, csrc/check.cuh trace).

Runs steps of C5 (--p, --n) without graphs and serialised, with SGM_TRACE_LAUNCH selecting the
traced sweep launch (ordinal among the process's sweep launches), then prints per-phase averages:
  producer: 0 issue start, 1 tile landed (FULL arrive)
  consumer warp 0: 2 wait start, 3 FULL passed, 4 phase A done, 5 tails barrier passed,
                   6 solve done (before store), 7 tile done
"""
import argparse
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_2302_04979_b200 as S  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--p", type=int, default=3)
ap.add_argument("--n", type=int, default=128)
ap.add_argument("--steps", type=int, default=6)
ap.add_argument("--opts", type=lambda s: int(s, 0), default=S.OPT_NO_GRAPH)
args = ap.parse_args()

pl = S.Plan((args.n,) * 3, args.p)
pl.set_options(args.opts)
g = torch.Generator(device="cuda").manual_seed(0)
d = torch.randn(pl.N_e, device="cuda", dtype=torch.float64, generator=g)
e = torch.zeros_like(d)
b = torch.randn(pl.N_h, device="cuda", dtype=torch.float64, generator=g)
h = torch.zeros_like(b)
st = torch.cuda.Stream()
with torch.cuda.stream(st):
    pl.step(d, e, b, h, 1e-3, args.steps, stream=st)
torch.cuda.synchronize()
if not hasattr(S._lib, "sgm_tune_trace") or "SGM_TRACE_LAUNCH" not in os.environ:
    print("product build or no SGM_TRACE_LAUNCH: steps run, no trace")
    sys.exit(0)
fn = S._lib.sgm_tune_trace
fn.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
buf = np.zeros(160 * 16 * 8, dtype=np.uint64)
rc = fn(buf.ctypes.data, buf.size)
if rc:
    sys.exit(f"no trace (rc {rc}): tuning build and SGM_TRACE_LAUNCH needed")
T = buf.reshape(160, 16, 8).astype(np.int64)
live = T[:, :, 3] > 0
t0 = T[T > 0].min()
R = np.where(T > 0, T - t0, -1) / 1e3  # us
ctas = np.nonzero(live.any(axis=1))[0]
ntile = live.sum(axis=1)[ctas]
print(f"launch {os.environ.get('SGM_TRACE_LAUNCH')}: {len(ctas)} CTAs, tiles per CTA {ntile.min()}..{ntile.max()}")
end = max(R[c, :, 7].max() for c in ctas)
print(f"span {end:.2f} us (first stamp to last tile done)")
first_full = np.array([R[c, 0, 3] for c in ctas])
first_issue = np.array([R[c, 0, 0] for c in ctas])
print(f"first issue at {first_issue.mean():.2f} us (max {first_issue.max():.2f}); first FULL at {first_full.mean():.2f} "
      f"(max {first_full.max():.2f})")
lastd = np.array([R[c, ntile[i] - 1, 7] for i, c in enumerate(ctas)])
print(f"CTA end: mean {lastd.mean():.2f} min {lastd.min():.2f} max {lastd.max():.2f}")
names = ["wait FULL", "phase A", "tails bar", "B-D", "store"]
for k, nm in enumerate(names):
    v = []
    for i, c in enumerate(ctas):
        for t in range(ntile[i]):
            v.append(R[c, t, 3 + k] - R[c, t, 2 + k])
    v = np.array(v)
    print(f"  consumer {nm:10s}: mean {v.mean():6.2f} us  median {np.median(v):6.2f}  max {v.max():6.2f}")
lat = []
for i, c in enumerate(ctas):
    for t in range(ntile[i]):
        if R[c, t, 1] >= 0 and R[c, t, 0] >= 0:
            lat.append(R[c, t, 1] - R[c, t, 0])
if lat:
    lat = np.array(lat)
    print(f"  producer issue->landed: mean {lat.mean():.2f} us median {np.median(lat):.2f} max {lat.max():.2f}")
per_tile = []
for i, c in enumerate(ctas):
    if ntile[i] >= 3:
        per_tile.append((R[c, ntile[i] - 1, 7] - R[c, 0, 7]) / (ntile[i] - 1))
if per_tile:
    print(f"  steady tile period: mean {np.mean(per_tile):.2f} us")
c = ctas[0]
print("CTA", c, "timeline (us):")
for t in range(ntile[0]):
    print("   ", " ".join(f"{x:7.2f}" for x in R[c, t]))
