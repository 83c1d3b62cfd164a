"""Anchor for ncu: culled SK-NR(32) iterations at C4 (dev tool)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np

import paper_2506_14780_b200 as sk
from paper_2506_14780_b200 import generators as G

c = G.config("C4")
p = sk.PointProblem(c.x, c.y, c.alpha, c.beta, c.epsilon)
p.set_culling(60.0)
w = sk.solve(p, tol=1e-300, max_iter=30, trace=False)
rng = np.random.default_rng(0)
V = np.linalg.qr(rng.standard_normal((c.n, c.ell)))[0] * np.sqrt(c.n)
b = sk.SpectralBasis(np.asfortranarray(V), np.asfortranarray(V), np.zeros(c.ell), c.epsilon)
r = sk.solve(p, tol=1e-300, max_iter=3, ell=c.ell, basis=b, init=(w.f, w.g), trace=False)
print("done", r.iterations)
