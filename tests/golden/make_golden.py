"""Generate the committed golden fixtures from the UNMODIFIED reference.

Runs in the build container only (needs oracle/_ref/libfewha_ref.so, compiled
in place from /root/reference by oracle/Makefile).  Re-run with

    make -C oracle ref && python tests/golden/make_golden.py

Each fixture (.npz) holds, for one preset:
  * derived geometry: layer/DM extents, active masks (finalize_geometry,
    geometry.hpp:366-377)
  * the Jacobi preconditioner (operators.hpp:367-425)
  * operator probes on seeded N(0,1) inputs: W^-1, W, P, P^T, Gamma, Gamma^T,
    apply_M, build_rhs, add_dm_slopes, fit_to_mirrors
  * a recorded closed loop exactly as run_bench drives it (bench.hpp:144-154):
    per frame the slopes fed to step and the resulting c, a^(1), rho.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
from oracle import RefOracle  # noqa: E402

PRESETS = {
    "mini": ("presets/mini.json", 8),
    "small_mcao": ("presets/small_mcao.json", 4),
}


def make(name, rel, frames, seed=1):
    path = os.path.join(ROOT, rel)
    r = RefOracle(path, threads=1)
    d = r.dims
    ext, dext, masks = r.geometry()
    rng = np.random.default_rng(1234)
    x = rng.standard_normal(d.n)
    wf = rng.standard_normal(d.Nw)
    m = rng.standard_normal(d.S)
    a = rng.standard_normal(d.A)
    out = dict(
        layer_extent=ext, dm_extent=dext, masks=masks,
        in_x=x, in_wf=wf, in_meas=m, in_a=a,
        winv=r.wavelet(x, True), wfwd=r.wavelet(x, False),
        P=r.propagate(x), PT=r.propagate_transpose(wf), G=r.sh(wf), GT=r.sh_transpose(m),
        M=r.apply_M(x), rhs=r.build_rhs(m), dm_slopes=r.add_dm_slopes(a, m), fit=r.fit(x),
    )
    r.build_preconditioner()
    out["precond"] = r.preconditioner()
    meas, c, am, rho, _ = r.record(seed, frames)
    out.update(loop_meas=meas, loop_c=c, loop_a=am, loop_rho=rho)
    st = r.get_state()
    out.update({"final_" + k: v for k, v in st.items()})
    dst = os.path.join(HERE, f"{name}.npz")
    np.savez_compressed(dst, **out)
    print(dst, os.path.getsize(dst), "bytes")


def make_geometry_only(name, rel):
    r = RefOracle(os.path.join(ROOT, rel), threads=1)
    ext, dext, masks = r.geometry()
    dst = os.path.join(HERE, f"{name}_geometry.npz")
    np.savez_compressed(dst, layer_extent=ext, dm_extent=dext, masks=masks)
    print(dst, os.path.getsize(dst), "bytes")


def make_filters():
    orders = {}
    for order in range(1, 11):
        n = 16
        rng = np.random.default_rng(order)
        x = rng.standard_normal((n, n))
        orders[f"x{order}"] = x
        orders[f"fwd{order}"] = RefOracle.wavelet_grid(order, x, False)
        orders[f"inv{order}"] = RefOracle.wavelet_grid(order, x, True)
    dst = os.path.join(HERE, "wavelet_orders.npz")
    np.savez_compressed(dst, **orders)
    print(dst, os.path.getsize(dst), "bytes")


if __name__ == "__main__":
    for k, (rel, frames) in PRESETS.items():
        make(k, rel, frames)
    make_geometry_only("elt_mcao84", "presets/elt_mcao84.json")
    make_filters()
