import sys, time, ctypes as C; sys.path.insert(0, '.')
import numpy as np, torch
import paper_2009_00946_b200 as fg
rec = fg.Reconstructor("presets/elt_mcao84_3dm.json"); rec.build_preconditioner()
st = torch.cuda.Stream(); torch.cuda.set_stream(st); rec.set_stream(st.cuda_stream)
d = rec.dims
pin_s = torch.from_numpy(np.random.default_rng(0).standard_normal(d.S) * 0.01).pin_memory()
pin_a = torch.zeros(d.A, dtype=torch.float64).pin_memory(); pin_r = torch.zeros(d.iters, dtype=torch.float64).pin_memory()
L = fg.lib(); dp = C.POINTER(C.c_double); nr = (C.c_int * 1)()
def T(f, n=300):
    for _ in range(20): f()
    ts = []
    for _ in range(n):
        torch.cuda.synchronize(); t = time.perf_counter(); f(); ts.append((time.perf_counter() - t) * 1e6)
    return f"p50 {np.percentile(ts, 50):.1f} us  min {np.min(ts):.1f}"
ps, pa, pr = C.cast(pin_s.data_ptr(), dp), C.cast(pin_a.data_ptr(), dp), C.cast(pin_r.data_ptr(), dp)
print("step(all outputs)     ", T(lambda: L.fewha_gpu_step(rec._h, ps, None, pa, pr, nr)))
print("step(dm only)         ", T(lambda: L.fewha_gpu_step(rec._h, ps, None, pa, None, None)))
print("step(no outputs)      ", T(lambda: L.fewha_gpu_step(rec._h, ps, None, None, None, None)))
print("step_device + sync    ", T(lambda: (rec.step_device(None), rec.sync())))
print("load_slopes(pinned)+sync", T(lambda: (L.fewha_gpu_load_slopes(rec._h, C.c_void_p(pin_s.data_ptr()), 0), rec.sync())))
