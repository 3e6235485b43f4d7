"""Throughput of batched engines (instances per engine B) on one GPU, graph-timed:
recon/s = B * frames / time, inputs resident, no flush (profiling aid).

    python tools/batch_sweep.py [--sizes 1,2,4,8,16,32,64] [--streams 1]
"""
import argparse
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2009_00946_b200 as fg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--preset", default=os.path.join(ROOT, "presets", "elt_mcao84_3dm.json"))
ap.add_argument("--sizes", default="1,2,4,8,16,32,64")
ap.add_argument("--total", type=int, default=64, help="instances per step (engines = total / B)")
ap.add_argument("--precision", type=int, default=64)
a = ap.parse_args()
for B in [int(x) for x in a.sizes.split(",")]:
    ne = max(1, a.total // B)
    engines, streams = [], []
    for e in range(ne):
        r = fg.Reconstructor(a.preset, precision=a.precision, batch=B)
        r.build_preconditioner()
        st = torch.cuda.Stream()
        r.set_stream(st.cuda_stream)
        s = torch.from_numpy(np.random.default_rng(e).standard_normal(r.dims.S * B) * 0.01).cuda()
        r.load_slopes_device(s.data_ptr())
        engines.append((r, s))
        streams.append(st)
    for r, _ in engines:
        for _ in range(3):
            r.step_device(None)
    torch.cuda.synchronize()
    K = 20
    for mode in ("serial", "concurrent"):
        main = torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(main)
        for st in streams:
            st.wait_event(e0)
        for _ in range(K):
            for i, (r, _) in enumerate(engines):
                if mode == "serial":
                    r.set_stream(streams[0].cuda_stream)
                else:
                    r.set_stream(streams[i].cuda_stream)
                r.step_device(None)
        for st in streams:
            ev = torch.cuda.Event()
            ev.record(st)
            main.wait_event(ev)
        e1.record(main)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / K
        print(f"B={B:3d} engines={ne:3d} {mode:10s}: {ms:7.3f} ms per {B * ne} instances -> "
              f"{B * ne * 1000.0 / ms:9.1f} recon/s", flush=True)
    for r, _ in engines:
        r.close()
