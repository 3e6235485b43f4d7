"""Per-rank phase stamps of one forward and one inverse cluster launch inside the
real frame graph (FEWHA_GRAPH_STAMPS=1): median over frames and layers of each
stamp, us after the launch's median programmatic-wait stamp (1).

    python tools/diag/rank_stamps.py [--slots 6 7] [--frames 20]
"""
import argparse
import os
import sys

import numpy as np

os.environ["FEWHA_GRAPH_STAMPS"] = "1"
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2009_00946_b200 as fg  # noqa: E402

if os.environ.get("FEWHA_LIB"):  # A/B of library builds
    fg.LIB_PATH = os.environ["FEWHA_LIB"]

ap = argparse.ArgumentParser()
ap.add_argument("--preset", default=os.path.join(ROOT, "presets", "elt_mcao84_3dm.json"))
ap.add_argument("--frames", type=int, default=20)
ap.add_argument("--slots", type=int, nargs="+", default=[6, 7])
a = ap.parse_args()
import torch  # noqa: E402

rec = fg.Reconstructor(a.preset, precision=64)
rec.build_preconditioner()
rec.phase_stamps(enable_only=True)
C = rec.plan_info()["cluster_ctas"]
s = np.random.default_rng(0).standard_normal(rec.dims.S) * 0.01
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
acc = {slot: [] for slot in a.slots}
for f in range(a.frames):
    flush.zero_()
    torch.cuda.synchronize()
    rec.step(s)
    st = rec.phase_stamps().astype(np.int64)
    if f < 2:
        continue
    for slot in a.slots:
        arr = st[slot]
        used = arr[:, 0] > 0
        nb = int(used.sum())
        blk = arr[:nb].astype(np.float64)
        if os.environ.get("FEWHA_STAMP_CLOCK"):  # SM cycles: relative to each CTA's own stamp 1
            rel = np.where(blk > 0, blk - blk[:, 1:2], np.nan)
        else:
            w = np.median(blk[:, 1][blk[:, 1] > 0])
            rel = np.where(blk > 0, (blk - w) / 1000.0, np.nan)
        acc[slot].append(rel)
for slot in a.slots:
    r = np.array(acc[slot])  # frames x blocks x 16
    nb = r.shape[1]
    print(f"slot {slot}: {nb} CTAs, cluster {C}; per rank (median over frames and layers), us after the median wait")
    ks = [k for k in range(16) if np.isfinite(r[:, :, k]).any()]
    print("  rank " + " ".join(f"{k:>6d}" for k in ks))
    for q in range(C):
        sel = r[:, q::C, :]
        print(f"  {q:4d} " + " ".join(f"{np.nanmedian(sel[:, :, k]):6.0f}" if os.environ.get("FEWHA_STAMP_CLOCK") else f"{np.nanmedian(sel[:, :, k]):6.2f}" if np.isfinite(sel[:, :, k]).any() else "     -"
                                     for k in ks))
