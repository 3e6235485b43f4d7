"""Stage-timing CSV in the reference's bench schema (bench.hpp:214-228):

    sweep_param,value,rep,step_time_us,stage1_us,stage2_us,stage3_us,pcg_us

    python tools/bench_csv.py --out profiles/r01_bench_stages.csv [--reps 50]

Sweeps the batch size (instances per frame) over --batches on the ELT MCAO-84
3-DM preset; each row is one frame with StepTelemetry on (device event nodes
around every launch): step_time_us = telemetry total.
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2009_00946_b200 as fg  # noqa: E402

HEADER = "sweep_param,value,rep,step_time_us,stage1_us,stage2_us,stage3_us,pcg_us"

ap = argparse.ArgumentParser()
ap.add_argument("--preset", default=os.path.join(ROOT, "presets", "elt_mcao84_3dm.json"))
ap.add_argument("--batches", default="1,8,64")
ap.add_argument("--reps", type=int, default=50)
ap.add_argument("--precision", type=int, default=64)
ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "bench_stages.csv"))
a = ap.parse_args()
rows = []
for B in [int(x) for x in a.batches.split(",")]:
    rec = fg.Reconstructor(a.preset, precision=a.precision, batch=B)
    rec.build_preconditioner()
    rec.enable_telemetry(True)
    s = np.random.default_rng(0).standard_normal(rec.dims.S * B) * 0.01
    for _ in range(3):
        rec.step(s, want_coeffs=False)
    for rep in range(a.reps):
        rec.step(s, want_coeffs=False)
        t = rec.last_telemetry()
        rows.append(f"batch,{B},{rep},{t['total_us']:.3f},{t['stage1_us']:.3f},{t['stage2_us']:.3f},"
                    f"{t['stage3_us']:.3f},{t['pcg_us']:.3f}")
    med = np.median([float(r.split(",")[3]) for r in rows[-a.reps:]])
    print(f"batch {B}: median step {med:.1f} us")
    rec.close()
os.makedirs(os.path.dirname(a.out), exist_ok=True)
with open(a.out, "w") as f:
    f.write(HEADER + "\n" + "\n".join(rows) + "\n")
print("wrote", a.out)
