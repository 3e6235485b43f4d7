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

if os.environ.get("FEWHA_SCHED"):  # experiment: CUDA host-sync scheduling before any context exists
    from cuda.bindings import runtime as _rt
    _flag = {"spin": _rt.cudaDeviceScheduleSpin, "yield": _rt.cudaDeviceScheduleYield,
             "block": _rt.cudaDeviceScheduleBlockingSync}[os.environ["FEWHA_SCHED"]]
    print("cudaSetDeviceFlags", _rt.cudaSetDeviceFlags(_flag))
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
# the bench's pattern: 16 different page-locked frames in rotation
ring = torch.from_numpy(np.random.default_rng(1).standard_normal((16, d.S)) * 0.01).pin_memory()
ring_p = [C.cast(ring[f].data_ptr(), dp) for f in range(16)]
kk = [0]


def rot():
    kk[0] += 1
    return L.fewha_gpu_step(rec._h, ring_p[kk[0] % 16], None, pa, pr, nr)


T("step(dm + rho), 16-frame ring", rot)

# the same ring in transparent-huge-page-backed memory registered with CUDA
import mmap  # noqa: E402

from cuda.bindings import runtime as rt  # noqa: E402

HP = 2 << 20
nbytes = 16 * d.S * 8
mm = mmap.mmap(-1, nbytes + 2 * HP, flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
base = np.frombuffer(mm, dtype=np.uint8)
off = (-base.ctypes.data) % HP
mm.madvise(mmap.MADV_HUGEPAGE, off, nbytes + HP - off if off else nbytes + HP)
hp = base[off:off + nbytes].view(np.float64).reshape(16, d.S)
hp[:] = ring.numpy()
print("thp:", open("/sys/kernel/mm/transparent_hugepage/enabled").read().strip(),
      "register:", rt.cudaHostRegister(hp.ctypes.data, nbytes, rt.cudaHostRegisterDefault)[0])
hp_p = [C.cast(hp[f].ctypes.data, dp) for f in range(16)]


def rot_hp():
    kk[0] += 1
    return L.fewha_gpu_step(rec._h, hp_p[kk[0] % 16], None, pa, pr, nr)


T("step(dm + rho), 16-frame THP ring", rot_hp)
with open("/proc/self/smaps_rollup") as f:
    print([ln.strip() for ln in f if "AnonHugePages" in ln])
T("step(dm only)", lambda: L.fewha_gpu_step(rec._h, ps, None, pa, None, None))
T("step(no outputs)", lambda: L.fewha_gpu_step(rec._h, ps, None, None, None, None))
T("step_device + sync", lambda: (rec.step_device(None), rec.sync()))
T("load_slopes(pinned) + sync", lambda: (L.fewha_gpu_load_slopes(rec._h, C.c_void_p(pin_s.data_ptr()), 0), rec.sync()))
T("sync only", lambda: rec.sync())
T("empty ctypes call", lambda: L.fewha_gpu_launches_per_step(rec._h))
