import sys; sys.path.insert(0, '.'); sys.path.insert(0, 'oracle')
import numpy as np
import paper_2009_00946_b200 as fg
from oracle import Oracle, rel_err
name = sys.argv[1] if len(sys.argv) > 1 else "small_mcao"
o = Oracle(f"presets/{name}.json"); o.build_preconditioner(); J = o.preconditioner()
if name == "small_mcao":
    m0 = np.load("tests/golden/small_mcao.npz")["loop_meas"][0]
else:
    rng = np.random.default_rng(1); m0 = o.sh(o.propagate(rng.standard_normal(o.dims.n)))
r32 = fg.Reconstructor(f"presets/{name}.json", precision=32)
n = o.dims.n; sides = [1 << j for j in o.g["layer_order"]]
coarse = np.cumsum([0] + [s*s for s in sides])[:-1]
L = len(sides)
ad0 = np.array([o.apply_M(np.eye(1, n, k).ravel())[k] for k in coarse])  # M e_0 (fitting ~0 + alpha d0)
def cg(apply, b):
    c = np.zeros(n); r = b.copy(); p = np.zeros(n); q = np.zeros(n)
    for it in range(4):
        zz = r/J; s = apply(zz); rho = r@zz; mu = s@zz
        if it == 0: beta = 0; alpha = rho/mu
        else: beta = rho/rho_old; alpha = rho/(mu - rho*beta/alpha_old)
        rho_old, alpha_old = rho, alpha
        p = zz + beta*p; q = s + beta*q; c = c + alpha*p; r = r - alpha*q
    return c
b64 = o.build_rhs(m0); c_ref = cg(o.apply_M, b64)
print("coarse |b64|/|b|", np.abs(b64[coarse]).max()/np.abs(b64).max(), "coarse share of c", np.linalg.norm(c_ref[coarse])/np.linalg.norm(c_ref))
def fix(v, z=None):
    v = v.copy()
    v[coarse] = 0.0 if z is None else ad0 * z[coarse]
    return v
b32 = r32.build_rhs(m0)
print("fp32 plain", rel_err(cg(r32.apply_M, b32), c_ref))
print("fp32 coarse-exact", rel_err(cg(lambda z: fix(r32.apply_M(z), z), fix(b32)), c_ref))
print("fp64 coarse-exact vs ref", rel_err(cg(lambda z: fix(o.apply_M(z), z), fix(b64)), c_ref))
