import sys, ctypes as C; sys.path.insert(0, '.')
import numpy as np
import paper_2009_00946_b200 as fg
L = fg.lib()
L.fewha_gpu_debug_bench_dwt.restype = C.c_float
L.fewha_gpu_debug_bench_dwt.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int]
for prec in (64, 32):
    rec = fg.Reconstructor("presets/elt_mcao84.json", precision=prec)
    rec.wavelet(np.random.default_rng(0).standard_normal(rec.dims.n), True)  # allocate ops workspace
    for inv in (1, 0):
        res = {"cluster": L.fewha_gpu_debug_bench_dwt(rec._h, 0, inv, 50, 256)}
        for thr in (256, 512, 1024):
            res[f"single{thr}"] = L.fewha_gpu_debug_bench_dwt(rec._h, 1, inv, 50, thr)
        print(prec, "inverse" if inv else "forward", {k: round(v * 1000, 2) for k, v in res.items()}, "us/launch (9 layers)")
