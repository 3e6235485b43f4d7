"""Breakdown of the end-to-end fewha_gpu_step call (pinned host slopes in,
a1 + rho out) into its parts, host wall clock per call (profiling aid).

    python tools/e2e_break.py [--preset P] [--flush]
"""
import argparse
import ctypes as C
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2009_00946_b200 as fg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--preset", default=os.path.join(ROOT, "presets", "elt_mcao84_3dm.json"))
ap.add_argument("--flush", action="store_true", help="write 256 MiB before every call (as bench.py)")
ap.add_argument("--n", type=int, default=300)
args = ap.parse_args()

rec = fg.Reconstructor(args.preset)
rec.build_preconditioner()
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
rec.set_stream(st.cuda_stream)
d = rec.dims
flush = torch.empty(256 << 18, dtype=torch.float32, device="cuda")
pin_s = torch.from_numpy(np.random.default_rng(0).standard_normal(d.S) * 0.01).pin_memory()
pin_a = torch.zeros(d.A, dtype=torch.float64).pin_memory()
pin_r = torch.zeros(d.iters, dtype=torch.float64).pin_memory()
L = fg.lib()
dp = C.POINTER(C.c_double)
nr = (C.c_int * 1)()
ps, pa, pr = C.cast(pin_s.data_ptr(), dp), C.cast(pin_a.data_ptr(), dp), C.cast(pin_r.data_ptr(), dp)


def T(name, f):
    for _ in range(20):
        f()
    ts = []
    for _ in range(args.n):
        if args.flush:
            flush.zero_()
        torch.cuda.synchronize()
        t = time.perf_counter()
        f()
        ts.append((time.perf_counter() - t) * 1e6)
    print(f"{name:28s} p50 {np.percentile(ts, 50):7.1f} us  mean {np.mean(ts):7.1f}  min {np.min(ts):7.1f}  "
          f"p99 {np.percentile(ts, 99):7.1f}")


T("step(dm + rho)", lambda: L.fewha_gpu_step(rec._h, ps, None, pa, pr, nr))
T("step(dm only)", lambda: L.fewha_gpu_step(rec._h, ps, None, pa, None, None))
T("step(no outputs)", lambda: L.fewha_gpu_step(rec._h, ps, None, None, None, None))
T("step_device + sync", lambda: (rec.step_device(None), rec.sync()))
T("load_slopes(pinned) + sync", lambda: (L.fewha_gpu_load_slopes(rec._h, C.c_void_p(pin_s.data_ptr()), 0), rec.sync()))
T("sync only", lambda: rec.sync())
T("empty ctypes call", lambda: L.fewha_gpu_launches_per_step(rec._h))
