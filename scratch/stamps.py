import sys; sys.path.insert(0, '.')
import numpy as np
import paper_2009_00946_b200 as fg
prec = int(sys.argv[1]) if len(sys.argv) > 1 else 64
rec = fg.Reconstructor("presets/elt_mcao84.json", precision=prec)
rec.build_preconditioner()
s = np.random.default_rng(0).standard_normal(rec.dims.S) * 0.01
for _ in range(3): rec.step(s)
rec.phase_stamps(enable_only=True)
for _ in range(3): prof = rec.profile_step()
st = rec.phase_stamps()
kinds = [k for k, _ in prof if k not in ("wfs", "wfs_rhs", "fit_control")]
ms = dict()
for slot, kind in enumerate(kinds):
    a = st[slot].astype(np.int64)
    used = a[:, 0] > 0
    a = a[used]
    t0 = a[:, 0].min()
    rel = np.where(a > 0, a - t0, -1)
    cols = [k for k in range(16) if (rel[:, k] >= 0).any()]
    summ = " ".join(f"{k}:{rel[:, k][rel[:, k] >= 0].max()/1000:.1f}" for k in cols)
    print(f"{slot:2d} {kind:9s} blocks={used.sum():3d} max-over-CTAs us since first start: {summ}")
print([(k, round(t * 1000, 1)) for k, t in prof])
