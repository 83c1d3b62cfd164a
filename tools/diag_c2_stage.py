import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import oracle_ref as O
import paper_2506_14780_b200 as sk
from paper_2506_14780_b200 import generators as G
inst = G.config("C2")
eps = list(inst.epsilons)
op = O.Instance(inst.alpha, inst.beta, eps[0], x=inst.x, y=inst.y, cost_div=1.0 / inst.cost_scale)
gp = sk.PointProblem(inst.x, inst.y, inst.alpha, inst.beta, eps[0], inst.cost_scale)
prev = O.solve(op, tol=1e-9)
basis = O.top_modes(op, prev["f"], prev["g"], inst.ell)
for s in range(1, 4):
    prev = O.solve(op.with_epsilon(eps[s]), tol=1e-9, ell=inst.ell, V=basis["vectors"], init=(prev["f"], prev["g"])) if s < 3 else prev
e = eps[3]
gp.set_epsilon(e)
sb = sk.SpectralBasis(basis["vectors"], basis["vectors_sym"], basis["rhos"], eps[0])
rg = sk.solve(gp, tol=1e-9, ell=inst.ell, basis=sb, init=(prev["f"], prev["g"]))
ro = O.solve(op.with_epsilon(e), tol=1e-9, ell=inst.ell, V=basis["vectors"], init=(prev["f"], prev["g"]))
for k in range(max(rg.iterations, ro["iterations"])):
    a = rg.trace[k] if k < len(rg.trace) else None
    b = ro["trace"][k] if k < len(ro["trace"]) else None
    print(k + 1, f"gap {a.marginal_error if a else float('nan'):.10e} {b[0] if b else float('nan'):.10e}",
          f"Q {a.semi_dual_value if a else 0:.17e} {b[2] if b else 0:.17e}", f"acc {int(a.newton_accepted) if a else -1}{b[4] if b else -1}")
