"""ncu target: a few top_modes sweeps at C3 size (dev tool)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import paper_2506_14780_b200 as sk
from paper_2506_14780_b200 import generators as G
inst = G.config("C3")
pw = sk.PointProblem(inst.x, inst.y, inst.alpha, inst.beta, inst.basis_eps, inst.cost_scale)
f0 = np.zeros(inst.n)
g0 = sk.ctransform_of_f(pw, f0)
t0 = time.time()
try:
    sk.top_modes(pw, f0, g0, inst.ell, max_power_iters=int(sys.argv[1]) if len(sys.argv) > 1 else 20)
except sk.EigensolverError as e:
    pass
print(f"top_modes sweeps wall {time.time()-t0:.3f}s")
