"""Eager frames of the ELT MCAO-84 reconstruction for ncu (one process, 1 GPU).

    ncu --metrics gpu__time_duration.sum --clock-control none --csv \
        --log-file profiles/<round>_launches.csv python tools/profile_frame.py
    ncu --set full --clock-control none --import-source on -k regex:k_adjoint -s 5 -c 1 \
        -o gpurun_out/adjoint python tools/profile_frame.py
Runs 2 warm-up frames then `--frames` profiled frames through
fewha_gpu_profile_step (eager launches, same kernels as the graph).
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2009_00946_b200 as fg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--preset", default=os.path.join(ROOT, "presets", "elt_mcao84_3dm.json"))
ap.add_argument("--precision", type=int, default=64)
ap.add_argument("--frames", type=int, default=2)
ap.add_argument("--batch", type=int, default=1)
a = ap.parse_args()
rec = fg.Reconstructor(a.preset, precision=a.precision, batch=a.batch)
rec.build_preconditioner()
s = np.random.default_rng(0).standard_normal(rec.dims.S * a.batch) * 0.01
for _ in range(2):
    rec.step(s)
for _ in range(a.frames):
    prof = rec.profile_step()
print({k: round(sum(t for kk, t in prof if kk == k) * 1000, 1) for k, _ in prof})
