import sys, os
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import numpy as np
import paper_2506_14780_b200 as sk
from paper_2506_14780_b200 import generators as G
from support import smooth_basis
inst = G.config("C4", n=2048, m=2048)
eps = 4e-3
gp = sk.PointProblem(inst.x, inst.y, inst.alpha, inst.beta, eps, inst.cost_scale)
V = np.asfortranarray(smooth_basis(inst.x, inst.alpha, 16))
basis = sk.SpectralBasis(V, V, np.zeros(16), eps)
for on in (True, False):
    sk.set_tensor_block_pass(on)
    rs = [sk.solve(gp, tol=1e-9, max_iter=3000, ell=16, basis=basis, trace=True, accept="stable") for _ in range(3)]
    accs = [[t.newton_accepted for t in r.trace] for r in rs]
    print("i8" if on else "fp64", [r.iterations for r in rs], "acc equal:", accs[0] == accs[1] == accs[2],
          "f bitwise:", all(np.array_equal(rs[0].f, r.f) for r in rs))
    r = sk.solve(gp, tol=1e-9, max_iter=5, trace=False)
    outs = [sk.restricted_derivatives(gp, r.f, basis) for _ in range(5)]
    print("  derivs bitwise:", all(np.array_equal(outs[0][1], o[1]) and np.array_equal(outs[0][0], o[0]) for o in outs))
