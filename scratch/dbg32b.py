import sys; sys.path.insert(0, '.'); sys.path.insert(0, 'oracle')
import numpy as np
import paper_2009_00946_b200 as fg
from oracle import Oracle, rel_err
name = sys.argv[1]
g = np.load(f"tests/golden/{name}.npz")
m0 = g["loop_meas"][0]
r64 = fg.Reconstructor(f"presets/{name}.json", precision=64)
r32 = fg.Reconstructor(f"presets/{name}.json", precision=32)
print("M op", rel_err(r32.apply_M(g["in_x"]), g["M"]), "rhs op", rel_err(r32.build_rhs(g["in_meas"]), g["rhs"]))
print("precond", rel_err(r32.preconditioner(), r64.preconditioner()))
a64 = r64.step(m0); a32 = r32.step(m0)
s64, s32 = r64.get_state(), r32.get_state()
for k in ("b", "r", "c", "p", "q"): print(k, rel_err(s32[k], s64[k]))
print("rho", r64.last_rho, r32.last_rho)
# one-iteration config
import json
j = json.load(open(f"presets/{name}.json")); j["solver"]["pcg_max_iter"] = 1
for prec in (64, 32):
    r = fg.Reconstructor(j, precision=prec); r.step(m0); st = r.get_state()
    print(prec, "1-iter c", st["c"][:4], "rho", r.last_rho)
