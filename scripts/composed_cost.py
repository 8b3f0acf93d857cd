"""Cost of one Yoshida (4th-order) composed step against three leapfrog steps at 128^3 p=3 (graph
replay on a dedicated stream, CUDA events)."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2302_04979_b200 as S  # noqa: E402
import synth  # noqa: E402

pl = S.Plan(128, 3)
d0, b0 = synth.normal(5, pl.N_e, pl.N_h)
d = torch.from_numpy(d0).cuda(); b = torch.from_numpy(b0).cuda()
e, h = torch.empty_like(d), torch.empty_like(b)
st = torch.cuda.Stream()
dt = 0.5 * 0.2020 / 128
a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
with torch.cuda.stream(st):
    pl.hodge_star(S.MASS_EPS, d, e, stream=st); pl.hodge_star(S.MASS_MU, b, h, stream=st)
    for fn, name in ((lambda: pl.step(d, e, b, h, dt, 3, stream=st), "3 leapfrog steps"),
                     (lambda: pl.step_composed(d, e, b, h, dt, S.YOSHIDA4, 1, stream=st), "1 Yoshida step")):
        for _ in range(5):
            fn()
        st.synchronize()
        a.record(st)
        for _ in range(50):
            fn()
        z.record(st)
        st.synchronize()
        print(f"{name}: {1e3 * a.elapsed_time(z) / 50:.1f} us")
