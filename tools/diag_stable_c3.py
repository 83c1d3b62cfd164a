"""Diagnose the stable-accept decisions of test_full_size_trajectory (BASELINE C3, full size):
K SK iterations from f = 0, then KN SK-NR steps with the smooth basis, both accept modes,
GPU trace next to the oracle's (dQ as tested, max step)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np

import oracle_ref as O
import paper_2506_14780_b200 as sk
from paper_2506_14780_b200 import generators as G
from support import smooth_basis

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
K, KN = (6, 6) if name == "C3" else (2, 4)
c = G.config(name)
gp = sk.PointProblem(c.x, c.y, c.alpha, c.beta, c.epsilon, c.cost_scale)
op = O.Instance(c.alpha, c.beta, c.epsilon, x=c.x, y=c.y, cost_div=1.0 / c.cost_scale)
ro = O.solve(op, tol=1e-300, max_iter=K)
V = smooth_basis(c.x, c.alpha, c.ell)
basis = sk.SpectralBasis(V, V, np.zeros(c.ell), c.epsilon)
init = (ro["f"], ro["g"])
for mode in ("stable", "literal"):
    ng = sk.solve(gp, tol=1e-300, max_iter=KN, ell=c.ell, basis=basis, init=init, accept=mode)
    with O.accept_mode(mode):
        no = O.solve(op, tol=1e-300, max_iter=KN, ell=c.ell, V=V, init=init)
    print(f"--- {name} {mode}: eps {c.epsilon}")
    for k, (tg, to) in enumerate(zip(ng.trace, no["trace"])):
        print(f"{k + 1}: gpu acc {tg.newton_accepted} Q {tg.semi_dual_value:.17g} err {tg.marginal_error:.6e} | "
              f"oracle acc {int(to[4])} Q {to[2]:.17g} err {to[0]:.6e} gain {to[5]:.6e} step {to[6]:.3e} "
              f"step/eps {to[6] / c.epsilon:.1f}")
    print("rel f", float(np.max(np.abs(ng.f - no["f"])) / np.max(np.abs(no["f"]))))
