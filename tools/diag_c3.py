"""Diagnose C3 SK trajectory: GPU vs oracle for K iterations (dev tool)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np

import oracle_ref as O
import paper_2506_14780_b200 as sk
from paper_2506_14780_b200 import generators as G

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 30
n = int(sys.argv[3]) if len(sys.argv) > 3 else None
inst = G.config(cfg, n=n, m=n)
gp = sk.PointProblem(inst.x, inst.y, inst.alpha, inst.beta, inst.epsilon, inst.cost_scale)
rg = sk.solve(gp, tol=1e-300, max_iter=K)
t0 = time.time()
op = O.Instance(inst.alpha, inst.beta, inst.epsilon, x=inst.x, y=inst.y, cost_div=1.0 / inst.cost_scale)
ro = O.solve(op, tol=1e-300, max_iter=K)
print(f"oracle {time.time()-t0:.1f}s")
for k in range(K):
    print(k + 1, f"{rg.trace[k].marginal_error:.10e} {ro['trace'][k][0]:.10e}")
print("rel f", np.max(np.abs(rg.f - ro["f"])) / np.max(np.abs(ro["f"])))
g = sk.ctransform_of_f(gp, ro["f"])
print("ctransform at oracle f rel", np.max(np.abs(g - O.ctransform_of_f(op, ro["f"]))) / np.max(np.abs(g)))
