"""Anchor for ncu: C4 with culling, 20 SK iterations from f = 0 (dev tool)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2506_14780_b200 as sk
from paper_2506_14780_b200 import generators as G

c = G.config("C4")
p = sk.PointProblem(c.x, c.y, c.alpha, c.beta, c.epsilon)
p.set_culling(60.0)
r = sk.solve(p, tol=1e-300, max_iter=int(sys.argv[1]) if len(sys.argv) > 1 else 20, trace=False)
print("iterations", r.iterations, sk.debug_counters(p))
