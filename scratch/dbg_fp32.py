import sys, os; sys.path.insert(0, '.'); sys.path.insert(0, 'oracle')
import numpy as np
import paper_2009_00946_b200 as fg
from oracle import Oracle, rel_err
g = np.load("tests/golden/small_mcao.npz")
m0 = g["loop_meas"][0]
o = Oracle("presets/small_mcao.json"); o.build_preconditioner(); J = o.preconditioner()
r64 = fg.Reconstructor("presets/small_mcao.json", precision=64)
r32 = fg.Reconstructor("presets/small_mcao.json", precision=32)
b_o = o.build_rhs(m0)
print("rhs64", rel_err(r64.build_rhs(m0), b_o), "rhs32", rel_err(r32.build_rhs(m0), b_o))
print("J32", rel_err(r32.preconditioner(), J))
z = b_o / J
print("M(z)64", rel_err(r64.apply_M(z), o.apply_M(z)), "M(z)32", rel_err(r32.apply_M(z), o.apply_M(z)))
# emulated CG with GPU fp32 operators
def cg(apply):
    n = b_o.size; c = np.zeros(n); r = b_o.copy(); p = np.zeros(n); q = np.zeros(n)
    for it in range(4):
        zz = r/J; s = apply(zz); rho = r@zz; mu = s@zz
        if it == 0: beta = 0; alpha = rho/mu
        else: beta = rho/rho_old; alpha = rho/(mu - rho*beta/alpha_old)
        rho_old, alpha_old = rho, alpha
        p = zz + beta*p; q = s + beta*q; c = c + alpha*p; r = r - alpha*q
    return c
c_ref = cg(o.apply_M); c32e = cg(r32.apply_M)
print("emulated CG with GPU fp32 M:", rel_err(c32e, c_ref), " golden vs cg64", rel_err(c_ref, g["loop_c"][0]))
for prec, rr in ((64, r64), (32, r32)):
    rr.reset()
    a = rr.step(m0)
    st = rr.get_state()
    print(prec, "step c", rel_err(st["c"], g["loop_c"][0]), "b", rel_err(st["b"], b_o), "rho", rr.last_rho, g["loop_rho"][0])
    for k in ("r", "p", "q"):
        print("   ", k, rel_err(st[k], g_st[k]) if False else np.linalg.norm(st[k]))
    print("   scalars", st["scalars"])
prof = r32.profile_step()
print(prof)
