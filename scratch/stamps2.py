import sys; sys.path.insert(0, '.')
import numpy as np
import paper_2009_00946_b200 as fg
rec = fg.Reconstructor("presets/elt_mcao84_3dm.json", precision=64)
rec.build_preconditioner()
s = np.random.default_rng(0).standard_normal(rec.dims.S) * 0.01
for _ in range(3): rec.step(s)
rec.phase_stamps(enable_only=True)
for _ in range(3): prof = rec.profile_step()
st = rec.phase_stamps()
kinds = [k for k, _ in prof if k not in ("fit_control",)]
for slot, kind in enumerate(kinds[:9]):
    a = st[slot].astype(np.int64); used = a[:, 0] > 0; a = a[used]; t0 = a[:, 0].min()
    rel = np.where(a > 0, a - t0, -1)
    cols = [k for k in range(16) if (rel[:, k] >= 0).any()]
    print(f"{slot:2d} {kind:9s} blocks={used.sum():3d} max: " + " ".join(f"{k}:{rel[:, k][rel[:, k] >= 0].max()/1000:.1f}" for k in cols)
          + " | median: " + " ".join(f"{k}:{np.median(rel[:, k][rel[:, k] >= 0])/1000:.1f}" for k in cols))
