"""Phase stamps of the whole-layer kernels in a batched frame (profiling aid):
per launch slot, median over CTAs of each stamp, us after the launch's first stamp.

    python tools/diag/wl_stamps.py [--batch 64] [--precision 64]
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
ap.add_argument("--batch", type=int, default=64)
ap.add_argument("--precision", type=int, default=64)
a = ap.parse_args()
rec = fg.Reconstructor(a.preset, precision=a.precision, batch=a.batch)
rec.build_preconditioner()
rec.phase_stamps(enable_only=True)
s = np.random.default_rng(0).standard_normal(rec.dims.S * a.batch) * 0.01
for _ in range(3):
    rec.step(s)
prof = rec.profile_step()
st = rec.phase_stamps().astype(np.float64)
kinds = [k for k, _ in prof]
slot = 0
for kind, ms in prof:
    if kind == "fit_control":
        continue  # (launched without a stamp slot)
    arr = st[slot]
    slot += 1
    if kind in ("wfs_rhs", "wfs"):
        continue
    used = arr[:, 0] > 0
    blk = arr[used]
    if not len(blk):
        continue
    t0 = blk[:, 0].min()
    med = [np.median(blk[:, k][blk[:, k] > 0] - t0) / 1000 if (blk[:, k] > 0).any() else np.nan for k in range(16)]
    span = [np.median((blk[:, k + 1] - blk[:, k])[(blk[:, k + 1] > 0) & (blk[:, k] > 0)]) / 1000
            if ((blk[:, k + 1] > 0) & (blk[:, k] > 0)).any() else np.nan for k in range(6)]
    print(f"{kind:10s} {ms * 1000:8.1f} us  CTAs {len(blk):5d}  per-CTA phase us: " +
          " ".join(f"{k}->{k + 1}:{v:.2f}" for k, v in enumerate(span) if np.isfinite(v)))
