"""Diagnostic: per-frame rel err of the GPU loop vs the oracle (fp64/fp32), and the
oracle's own spread under input jitter (its conditioning).  Prints a table."""
import os, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
for p in (ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")):
    sys.path.insert(0, p)
import numpy as np
import paper_2009_00946_b200 as fg
from oracle import Oracle, rel_err
from test_gpu_parity import smooth_layers, noisy_slopes

name, frames, prec = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
batch = int(sys.argv[4]) if len(sys.argv) > 4 else 1
path = os.path.join(ROOT, "presets", name + ".json")
os_ = [Oracle(path) for _ in range(batch)]
for o in os_:
    o.build_preconditioner()
g = fg.Reconstructor(path, precision=prec, batch=batch)
lay = [smooth_layers(os_[0], 3 + i) for i in range(batch)]
closed = os_[0].g["loop_closed"]
worst = 0
for k in range(frames):
    ss, outs = [], []
    for i, o in enumerate(os_):
        st = o.get_state()
        s = noisy_slopes(os_[0], lay[i], 100 + k + 1000 * i, st["a_prev2"] if closed else None)
        ss.append(s)
        outs.append(o.step(s))
    a = g.step(np.stack(ss) if batch > 1 else ss[0])
    cs = g.coeffs()
    for i in range(batch):
        ai = a[i] if batch > 1 else a
        ci = cs[i] if batch > 1 else cs
        ri = g.last_rho[i] if batch > 1 else g.last_rho
        e = (rel_err(ci, outs[i][0]), rel_err(ai, outs[i][1]), rel_err(ri, outs[i][2]))
        print(k, i, "c %.2e a %.2e rho %.2e" % e, flush=True)
