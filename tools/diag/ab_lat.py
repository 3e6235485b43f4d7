"""A/B frame latency of library builds in one process each (profiling aid):
the bench's device-resident method (slopes loaded outside timing, 256 MiB L2
flush, CUDA events around each graph launch), 600 frames, p50 / p99.

    FEWHA_LIB=<path to libfewha_gpu.so> python tools/diag/ab_lat.py [--preset P] [--batch B] [--precision 64]
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2009_00946_b200 as fg  # noqa: E402

if os.environ.get("FEWHA_LIB"):
    fg.LIB_PATH = os.environ["FEWHA_LIB"]
ap = argparse.ArgumentParser()
ap.add_argument("--preset", default=os.path.join(ROOT, "presets", "elt_mcao84_3dm.json"))
ap.add_argument("--frames", type=int, default=600)
ap.add_argument("--batch", type=int, default=1)
ap.add_argument("--precision", type=int, default=64)
a = ap.parse_args()
import torch  # noqa: E402

dev = torch.device("cuda:0")
rec = fg.Reconstructor(a.preset, precision=a.precision, batch=a.batch)
rec.build_preconditioner()
S = rec.dims.S
rng = np.random.default_rng(1)
stream = torch.from_numpy(rng.standard_normal((8, a.batch * S)) * 0.01).to(dev)
st = torch.cuda.Stream(dev)
torch.cuda.set_stream(st)
rec.set_stream(st.cuda_stream)
flush = torch.empty((256 << 20) // 4, dtype=torch.float32, device=dev)
for k in range(10):
    rec.load_slopes_device(stream[k % 8].data_ptr())
    rec.step_device(None)
rec.sync()
starts = [torch.cuda.Event(enable_timing=True) for _ in range(a.frames)]
ends = [torch.cuda.Event(enable_timing=True) for _ in range(a.frames)]
for k in range(a.frames):
    rec.load_slopes_device(stream[k % 8].data_ptr())
    if a.batch == 1:
        flush.zero_()
    starts[k].record(st)
    rec.step_device(None)
    ends[k].record(st)
torch.cuda.synchronize(dev)
ms = np.array([s.elapsed_time(e) for s, e in zip(starts, ends)])
tag = os.path.basename(os.path.dirname(fg.LIB_PATH))
print(f"{tag:10s} batch {a.batch} fp{a.precision}: p50 {np.percentile(ms, 50):.4f} ms  p99 {np.percentile(ms, 99):.4f} ms"
      f"  ({a.batch / np.percentile(ms, 50) * 1000:.0f} recon/s)", flush=True)
