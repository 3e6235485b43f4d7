"""Overlapped timeline of REAL graph frames (programmatic launch on): every
launch's phase stamps (%globaltimer) recorded from inside the captured frame
graph (FEWHA_GRAPH_STAMPS=1), relative to the frame's first stamp.

    python tools/graph_timeline.py [--preset P] [--frames N]

Per launch: start = first CTA's entry, wait = median CTA past the programmatic
wait (stamp 1, or 12 for the gather), end = last CTA's final stamp (us).
"""
import argparse
import os
import sys

import numpy as np

os.environ["FEWHA_GRAPH_STAMPS"] = "1"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2009_00946_b200 as fg  # noqa: E402

if os.environ.get("FEWHA_LIB"):  # A/B of library builds
    fg.LIB_PATH = os.environ["FEWHA_LIB"]

ap = argparse.ArgumentParser()
ap.add_argument("--preset", default=os.path.join(ROOT, "presets", "elt_mcao84_3dm.json"))
ap.add_argument("--frames", type=int, default=20)
a = ap.parse_args()
import torch  # noqa: E402

rec = fg.Reconstructor(a.preset, precision=64)
rec.build_preconditioner()
rec.phase_stamps(enable_only=True)  # allocate before the graph is captured
s = np.random.default_rng(0).standard_normal(rec.dims.S) * 0.01
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
rows = []
for f in range(a.frames):
    flush.zero_()
    torch.cuda.synchronize()
    rec.step(s)
    st = rec.phase_stamps().astype(np.int64)
    used = [slot for slot in range(32) if (st[slot, :, 0] > 0).any()]
    t0 = min(st[slot][st[slot, :, 0] > 0, 0].min() for slot in used)
    fr = []
    for slot in used:
        arr = st[slot][st[slot, :, 0] > 0]
        start = (arr[:, 0].min() - t0) / 1000
        wcol = 12 if arr[:, 12].max() > 0 else 1
        wait = (np.median(arr[:, wcol][arr[:, wcol] > 0]) - t0) / 1000 if (arr[:, wcol] > 0).any() else np.nan
        last = max(k for k in range(12) if (arr[:, k] > 0).any())
        end = (arr[:, last].max() - t0) / 1000
        # every stamp: median over CTAs (us since the frame's first stamp)
        ph = [((np.median(arr[:, k][arr[:, k] > 0]) - t0) / 1000 if (arr[:, k] > 0).any() else np.nan) for k in range(16)]
        fr.append((slot, start, wait, end, *ph))
    rows.append(fr)
med_all = np.nanmedian(np.array([[x[1:] for x in fr] for fr in rows[2:]]), axis=0)
med = med_all[:, :3]
kinds = ["wfs_rhs", "gather", "fwd_rhs"] + ["inv", "wfs", "gather", "fwd"] * 4 + ["inv_fit"]
print("slot kind       start   wait    end   (us, median of frames; fit_control has no stamps)")
prev_end = 0.0
for i, (stt, w, e) in enumerate(med):
    k = kinds[i] if i < len(kinds) else "?"
    phs = " ".join(f"{j}:{v:.1f}" for j, v in enumerate(med_all[i, 3:]) if np.isfinite(v))
    print(f"{i:3d}  {k:8s} {stt:7.1f} {w:7.1f} {e:7.1f}   (+{e - prev_end:5.1f})   {phs}")
    prev_end = e
