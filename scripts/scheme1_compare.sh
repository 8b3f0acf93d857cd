python -m pytest tests -m gpu -q -x 2>&1 | tail -1
for SC in 2 1; do python bench.py --config c3 --scheme $SC --steps 10 --warmup 3 --no-cpu --no-e2e | python -c "import json,sys; d=json.load(sys.stdin); print('c3 scheme $SC', d['value'], d['ms_per_step'], {k:round(1e3*v['ms_per_launch'],1) for k,v in d['kernels'].items()})"; done
SGM_PCG_ITERS=20 python bench.py --config c3 --scheme 1 --steps 10 --warmup 3 --no-cpu --no-e2e | python -c "import json,sys; d=json.load(sys.stdin); print('c3 scheme 1 pcg20', d['ms_per_step'])"
python - <<'PY'
import numpy as np, torch, sys
sys.path.insert(0,'.')
import paper_2302_04979_b200 as S, synth
from oracle import workloads as W
p, n = 3, 48
ctrl = W.interpolate_map(p, n, W.c3_map)
for sc in (2, 1):
    pl = S.Plan(n, p, geom_ctrl=ctrl)
    X = pl.qp_coords(); c_eps, _ = synth.c3_centres()
    pl.set_material(S.EPS, np.where(np.linalg.norm(X - c_eps, axis=1) < 0.25, 4.0, 1.0))
    pl.set_scheme(sc)
    x = torch.from_numpy(synth.rng(100).standard_normal(pl.N_e)).cuda()
    e = torch.empty(pl.N_e, dtype=torch.float64, device="cuda"); b = torch.empty(pl.N_h, dtype=torch.float64, device="cuda"); h = torch.empty_like(b)
    out = torch.zeros(2, dtype=torch.float64, device="cuda")
    pl.cfl(x, e, b, h, out, 200); torch.cuda.synchronize(); print("c3 cfl scheme", sc, out.tolist())
PY
