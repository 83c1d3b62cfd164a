"""C4 culled SK-NR(32) iteration time (bench_iterations with a random orthonormal basis)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2506_14780_b200 as sk
from paper_2506_14780_b200 import generators as G
c = G.config("C4")
p = sk.PointProblem(c.x, c.y, c.alpha, c.beta, c.epsilon)
p.set_culling(60.0)
V = np.linalg.qr(np.random.default_rng(0).standard_normal((c.n, c.ell)))[0] * np.sqrt(c.n)
b = sk.SpectralBasis(np.asfortranarray(V), np.asfortranarray(V), np.zeros(c.ell), c.epsilon)
ms, k = sk.bench_iterations(p, c.ell, b, iters=10, warmup=2, flush_l2=True)
print("culled SK-NR(32) iteration ms", ms)
