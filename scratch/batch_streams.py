import sys, time; sys.path.insert(0, '.')
import numpy as np, torch
import paper_2009_00946_b200 as fg
P = "presets/elt_mcao84_3dm.json"
def run(nstreams, per, reps=20):
    recs, sts = [], []
    for i in range(nstreams):
        r = fg.Reconstructor(P, batch=per); r.build_preconditioner()
        st = torch.cuda.Stream(); r.set_stream(st.cuda_stream)
        s = np.random.default_rng(i).standard_normal(r.dims.S * per) * 0.01
        r.load_slopes(s)
        recs.append(r); sts.append(st)
    for _ in range(3):
        for r in recs: r.step_device(None)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        for r in recs: r.step_device(None)
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t) * 1e3 / reps
    tot = nstreams * per
    print(f"{nstreams} streams x batch {per}: {ms:.3f} ms per round -> {tot * 1000 / ms:.0f} recon/s")
    for r in recs: r.close()
for ns, per in [(1, 64), (2, 32), (4, 16), (8, 8), (16, 4), (4, 32), (8, 16), (1, 128)]:
    run(ns, per)
