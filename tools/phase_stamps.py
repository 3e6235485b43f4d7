"""Per-phase %globaltimer stamps of one eager ELT frame (profiling aid): for every
launch, the median / max over CTAs of each stamp (us since the launch's first CTA).

    python tools/phase_stamps.py [--preset P]          (FEWHA_FUSE=1: merged kernels)
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
ap.add_argument("--launches", type=int, default=9)
a = ap.parse_args()
rec = fg.Reconstructor(a.preset, precision=64)
rec.build_preconditioner()
s = np.random.default_rng(0).standard_normal(rec.dims.S) * 0.01
for _ in range(3):
    rec.step(s)
rec.phase_stamps(enable_only=True)
for _ in range(3):
    prof = rec.profile_step()
st = rec.phase_stamps()
print("launch ms:", " ".join(f"{k}:{t * 1000:.1f}" for k, t in prof[: a.launches + 2]))
for slot, (kind, _) in enumerate(prof[: a.launches]):
    arr = st[slot].astype(np.int64)
    used = arr[:, 0] > 0
    if not used.any():
        continue
    arr = arr[used]
    t0 = arr[:, 0].min()
    rel = np.where(arr > 0, arr - t0, -1)
    cols = [k for k in range(16) if (rel[:, k] >= 0).any()]
    med = " ".join(f"{k}:{np.median(rel[:, k][rel[:, k] >= 0]) / 1000:.1f}" for k in cols)
    mx = " ".join(f"{k}:{rel[:, k][rel[:, k] >= 0].max() / 1000:.1f}" for k in cols)
    print(f"{slot:2d} {kind:12s} blocks={used.sum():3d} median: {med} | max: {mx}")
