import sys, json, os; sys.path.insert(0, '.'); sys.path.insert(0, 'tests'); sys.path.insert(0, 'oracle')
import numpy as np
import paper_2009_00946_b200 as fg
from oracle import Oracle, rel_err
from test_gpu_parity import TRANSFORM_VARIANTS, _variant, smooth_layers, noisy_slopes
import pathlib, tempfile
tmp = pathlib.Path(tempfile.mkdtemp())
for case in sorted(TRANSFORM_VARIANTS):
    base, orders, wav = TRANSFORM_VARIANTS[case]
    path = _variant(tmp, base, case, orders, wav)
    g = fg.Reconstructor(path, precision=64); o = Oracle(path); o2 = Oracle(path)
    rng = np.random.default_rng(5); x = rng.standard_normal(o.dims.n); m = rng.standard_normal(o.dims.S)
    print(case, "M", rel_err(g.apply_M(x), o.apply_M(x)), "rhs", rel_err(g.build_rhs(m), o.build_rhs(m)))
    o.build_preconditioner(); g.build_preconditioner(); o2.build_preconditioner()
    print("  precond", rel_err(np.array(g.preconditioner()), np.array(o.preconditioner())) if hasattr(g,'preconditioner') else '')
    lay = smooth_layers(o, 3)
    for k in range(3):
        s = noisy_slopes(o, lay, 100 + k, o.get_state()["a_prev2"])
        a_g = g.step(s); c_o, a_o, rho_o = o.step(s)
        c_p, a_p, _ = o2.step(s * (1 + 1e-15 * np.random.default_rng(k).standard_normal(s.shape)))
        cg = g.coeffs()
        offs = np.cumsum([0] + [4 ** J for J in o.g["layer_order"]])
        per = [float(np.linalg.norm(cg[offs[i]:offs[i+1]] - c_o[offs[i]:offs[i+1]]) / np.linalg.norm(c_o)) for i in range(len(offs) - 1)]
        print(f"  frame {k}: c {rel_err(cg, c_o):.2e} a {rel_err(a_g, a_o):.2e} rho {rel_err(g.last_rho, rho_o):.2e} | oracle self-sens c {rel_err(c_p, c_o):.2e}; per-layer {['%.1e'%v for v in per]}")
        d = np.abs(cg - c_o); i = int(np.argmax(d)); print("    worst idx", i, cg[i], c_o[i])
