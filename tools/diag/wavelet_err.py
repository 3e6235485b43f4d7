"""Accuracy of the device layer transforms against an extended-precision
evaluation of the reference's algorithm (wavelet.hpp:115-196 in long double),
next to the reference's own fp64 rounding (the C oracle, bitwise the reference).

    FEWHA_LIB=<path to libfewha_gpu.so> python tools/diag/wavelet_err.py [preset]

Inputs: closed-loop coefficient vectors c (inverse) and their nodal images
(forward) from the oracle on noisy slopes.  Prints max|err| / max|x| per layer
(worst layer) and the relative L2 error of the whole vector.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2009_00946_b200 as fg  # noqa: E402

if os.environ.get("FEWHA_LIB"):
    fg.LIB_PATH = os.environ["FEWHA_LIB"]
from oracle import Oracle  # noqa: E402
from test_gpu_parity import noisy_slopes, smooth_layers  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "elt_mcao84_3dm"
path = os.path.join(ROOT, "presets", name + ".json")
o = Oracle(path)
g = fg.Reconstructor(path)


def filters(order):
    tab = os.path.join(ROOT, "paper_2009_00946_b200", "csrc", "daubechies_table.h")
    txt = open(tab).read().split("=", 1)[1].split(";", 1)[0]
    nums = [float(t) for t in txt.replace("{", " ").replace("}", " ").replace(",", " ").split()
            if t[:1] in "-0123456789" and ("." in t or "e" in t)]
    off = sum(2 * k for k in range(1, order))
    f = np.array(nums[off:off + 2 * order], dtype=np.longdouble)
    return f


def smat(s, taps):
    h = s // 2
    m = np.zeros((s, h), dtype=np.longdouble)
    for i in range(h):
        for k, t in enumerate(taps):
            m[(2 * i + k) % s, i] += t
    return m


def inverse_ld(X, lo_t, hi_t):
    X = X.astype(np.longdouble).copy()
    n = X.shape[0]
    s = 2
    while s <= n:
        h = s // 2
        Sl, Sh = smat(s, lo_t), smat(s, hi_t)
        B = X[:s, :s].copy()
        B = Sl @ B[:h, :] + Sh @ B[h:, :]
        B = B[:, :h] @ Sl.T + B[:, h:] @ Sh.T
        X[:s, :s] = B
        s *= 2
    return X


def forward_ld(X, lo_t, hi_t):
    X = X.astype(np.longdouble).copy()
    s = X.shape[0]
    while s >= 2:
        Sl, Sh = smat(s, lo_t), smat(s, hi_t)
        B = X[:s, :s].copy()
        B = np.concatenate([B @ Sl, B @ Sh], axis=1)
        B = np.concatenate([Sl.T @ B, Sh.T @ B], axis=0)
        X[:s, :s] = B
        s //= 2
    return X


import json  # noqa: E402

cfg = json.load(open(path))
order = cfg.get("wavelet_order", 3)
lo_t = filters(order)
hi_t = np.array([(1 if k % 2 == 0 else -1) * lo_t[len(lo_t) - 1 - k] for k in range(len(lo_t))], dtype=np.longdouble)
d = g.dims
sides = [2 ** lay_["grid_order"] for lay_ in cfg["layers"]]
assert sum(S * S for S in sides) == d.n
lay = smooth_layers(o, 3)
worst = {}
for k in range(4):
    s = noisy_slopes(o, lay, 100 + k, o.get_state()["a_prev2"])
    c, _, _ = o.step(s)
    for inv in (True, False):
        x = c if inv else o.wavelet(c, True)
        ref = o.wavelet(x, inv)
        gpu = g.wavelet(x, inv)
        ex = np.zeros(d.n, dtype=np.longdouble)
        off = 0
        for S in sides:
            blk = x[off:off + S * S].reshape(S, S)
            ex[off:off + S * S] = (inverse_ld if inv else forward_ld)(blk, lo_t, hi_t).ravel()
            off += S * S
        for tag, v in (("ref", ref), ("gpu", gpu)):
            e = np.abs(v.astype(np.longdouble) - ex)
            rel = float(np.sqrt((e ** 2).sum() / (ex ** 2).sum()))
            mx = float(e.max() / np.abs(ex).max())
            key = ("inv" if inv else "fwd", tag)
            worst[key] = max(worst.get(key, (0, 0)), (rel, mx))
        e = float(np.linalg.norm(gpu - ref) / np.linalg.norm(ref))
        worst[("inv" if inv else "fwd", "gpu-ref")] = max(worst.get(("inv" if inv else "fwd", "gpu-ref"), (0, 0)), (e, 0))
for k, v in sorted(worst.items()):
    print(f"{k[0]} {k[1]:8s} relL2 {v[0]:.3e}  max/max {v[1]:.3e}")
