import os, sys
import numpy as np
sys.path.insert(0, "/root/repo")
import paper_2506_14780_b200 as sk
from paper_2506_14780_b200 import generators as G
NN = 601
inst = G.config("C1", n=NN, m=433)
a = np.full(NN, 1 / NN); b = np.full(433, 1 / 433)
mk = lambda: sk.PointProblem(inst.x, inst.y, a, b, inst.epsilon)
for K in (1, 2, 3):
    out = sk.run_emulated_shards(mk, 8, lambda p: sk.solve(p, tol=1e-9, max_iter=K))
    print(K, [float(np.max(np.abs(o.g - out[0].g))) for o in out], [float(np.max(np.abs(o.f - out[0].f))) for o in out],
          [o.trace[-1].marginal_error for o in out][-2:])
