"""Per-iteration comparison GPU vs oracle for C1 SK-NR (diagnostic)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np

import oracle_ref as O
import paper_2506_14780_b200 as sk
from paper_2506_14780_b200 import generators as G

inst = G.config("C1")
gp = sk.PointProblem(inst.x, inst.y, inst.alpha, inst.beta, inst.epsilon)
op = O.Instance(inst.alpha, inst.beta, inst.epsilon, x=inst.x, y=inst.y)
w = O.solve(op.with_epsilon(inst.basis_eps), tol=1e-9)
b = O.top_modes(op.with_epsilon(inst.basis_eps), w["f"], w["g"], inst.ell)
sb = sk.SpectralBasis(b["vectors"], b["vectors_sym"], b["rhos"], inst.basis_eps)
rg = sk.solve(gp, tol=1e-9, ell=inst.ell, basis=sb, init=(w["f"], w["g"]))
ro = O.solve(op, tol=1e-9, ell=inst.ell, V=b["vectors"], init=(w["f"], w["g"]))
print("iters", rg.iterations, ro["iterations"])
for k, (tg, to) in enumerate(zip(rg.trace, ro["trace"])):
    print(f"{k+1:3d} gap {tg.marginal_error:.6e} {to[0]:.6e}  Q {tg.semi_dual_value:.17e} {to[2]:.17e} "
          f"dQ {tg.semi_dual_value-to[2]:+.2e} acc {int(tg.newton_accepted)}{int(to[4])}")
print("rel f", np.max(np.abs(rg.f - ro["f"])) / np.max(np.abs(ro["f"])))
