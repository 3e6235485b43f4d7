import sys, time; sys.path.insert(0, '.')
import numpy as np, torch
import paper_2009_00946_b200 as fg
rec = fg.Reconstructor("presets/elt_mcao84_3dm.json")
rec.build_preconditioner()
S = rec.dims.S
s = np.random.default_rng(0).standard_normal(S) * 0.01
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
rec.set_stream(st.cuda_stream)
for _ in range(5): rec.step(s)
def wall(f, n=50):
    ts = []
    for _ in range(n):
        torch.cuda.synchronize(); t = time.perf_counter(); f(); ts.append((time.perf_counter() - t) * 1e3)
    return np.percentile(ts, 50), np.min(ts)
print("step() host API       p50/min ms", wall(lambda: rec.step(s, want_coeffs=False)))
print("step_device+sync      p50/min ms", wall(lambda: (rec.step_device(None), rec.sync())))
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ts = []
for _ in range(50):
    ev0.record(st); rec.step_device(None); ev1.record(st); torch.cuda.synchronize(); ts.append(ev0.elapsed_time(ev1))
print("graph (events)        p50/min ms", np.percentile(ts, 50), np.min(ts))
ev0.record(st)
for _ in range(100): rec.step_device(None)
ev1.record(st); torch.cuda.synchronize()
print("graph back-to-back    ms/frame", ev0.elapsed_time(ev1) / 100)
prof = rec.profile_step()
tot = sum(t for _, t in prof)
print("eager profile total ms", tot)
agg = {}
for k, t in prof: agg[k] = agg.get(k, 0) + t
print({k: round(v * 1000, 1) for k, v in agg.items()})
