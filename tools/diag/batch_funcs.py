"""Per-function times inside the batch frame graph (bench.py graph_function_profile:
event-record nodes between launches) next to the plain graph p50 (profiling aid).

    python tools/diag/batch_funcs.py [--batch 64] [--precision 64]
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2009_00946_b200 as fg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--preset", default=bench.DEFAULT_PRESET)
ap.add_argument("--batch", type=int, default=64)
ap.add_argument("--precision", type=int, default=64)
ap.add_argument("--tag", default="")
a = ap.parse_args()
import torch  # noqa: E402

dev = torch.device("cuda:0")
rec = fg.Reconstructor(a.preset, precision=a.precision, batch=a.batch)
rec.build_preconditioner()
d = bench.preset_dims(a.preset)
rng = np.random.default_rng(1)
stream = torch.from_numpy(rng.standard_normal((4, a.batch * rec.dims.S)) * 0.01).to(dev)
st = torch.cuda.Stream(dev)
torch.cuda.set_stream(st)
rec.set_stream(st.cuda_stream)
for k in range(5):
    rec.load_slopes_device(stream[k % 4].data_ptr())
    rec.step_device(None)
rec.sync()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(21)]
ev[0].record(st)
for k in range(20):
    rec.load_slopes_device(stream[k % 4].data_ptr())
    rec.step_device(None)
    ev[k + 1].record(st)
torch.cuda.synchronize(dev)
ms = np.array([ev[k].elapsed_time(ev[k + 1]) for k in range(20)])
prof, fms = bench.graph_function_profile(rec, 3, lambda f: rec.load_slopes_device(stream[f % 4].data_ptr()), d, 8,
                                         batch=a.batch)
print(f"{a.tag:12s} graph p50 {np.median(ms):.4f} ms | telemetry frame {fms:.4f} ms | " +
      " ".join(f"{k}:{v['launch_ms'] * 1000:.1f}us" for k, v in sorted(prof.items(), key=lambda kv: -kv[1]['share'])),
      flush=True)
