import sys, time, os; sys.path.insert(0, '.'); sys.path.insert(0, 'oracle')
import numpy as np, torch
import paper_2009_00946_b200 as fg
from oracle import Oracle, rel_err
prec = int(sys.argv[1]) if len(sys.argv) > 1 else 64
rec = fg.Reconstructor("presets/elt_mcao84.json", precision=prec)
print("launches/step", rec.launches_per_step())
rec.build_preconditioner()
S = rec.dims.S
s = np.random.default_rng(0).standard_normal(S) * 0.01
st = torch.cuda.Stream(); torch.cuda.set_stream(st); rec.set_stream(st.cuda_stream)
for _ in range(5): rec.step(s)
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ts = []
for _ in range(50):
    ev0.record(st); rec.step_device(None); ev1.record(st); torch.cuda.synchronize(); ts.append(ev0.elapsed_time(ev1))
print("graph (events) p50/min ms", np.percentile(ts, 50), np.min(ts))
ev0.record(st)
for _ in range(100): rec.step_device(None)
ev1.record(st); torch.cuda.synchronize()
print("graph back-to-back ms/frame", ev0.elapsed_time(ev1) / 100)
# parity vs oracle, 3 frames
o = Oracle("presets/elt_mcao84.json"); g2 = fg.Reconstructor("presets/elt_mcao84.json", precision=prec)
rng = np.random.default_rng(1)
for k in range(3):
    m = rng.standard_normal(S) * 0.1
    c_o, a_o, r_o = o.step(m); a_g = g2.step(m)
    print("frame", k, "rel err c", rel_err(g2.coeffs(), c_o), "a", rel_err(a_g, a_o), "rho", rel_err(g2.last_rho, r_o))
