import sys; sys.path.insert(0, '.')
import numpy as np
import paper_2009_00946_b200 as fg
rec = fg.Reconstructor("presets/elt_mcao84.json", precision=int(sys.argv[1]) if len(sys.argv) > 1 else 64)
rec.build_preconditioner()
s = np.random.default_rng(0).standard_normal(rec.dims.S) * 0.01
for _ in range(3): rec.step(s)
rec.phase_stamps(enable_only=True)
for _ in range(3): prof = rec.profile_step()
st = rec.phase_stamps().reshape(-1)[: 4096 * 32].reshape(4096, 32).astype(np.int64)
used = st[:, 0] > 0
a = st[used]
t0 = a[:, 0].min()
names = ["start", "rhs tiles", "bar", "fwd rhs", "inv0", "bar"] + sum([[f"it{i} tiles", "bar", f"it{i} fwd", "bar", f"it{i} inv", "bar"] for i in range(4)], [])
cols = [k for k in range(32) if (a[:, k] > 0).all()]
prev = 0
for k in cols:
    mx = (a[:, k] - t0).max() / 1000
    print(f"{k:2d} {names[k] if k < len(names) else '?':10s} max {mx:7.1f} us  (+{mx - prev:5.1f})  min {(a[:, k] - t0).min()/1000:7.1f}")
    prev = mx
print(prof)
