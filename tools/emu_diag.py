"""Per-rank agreement of the emulated sharded solve (dev tool)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_14780_b200 as sk
from paper_2506_14780_b200 import generators as G

NN = int(os.environ.get("NN", "601"))
inst = G.config("C1", n=NN, m=433)
a = np.full(NN, 1 / NN)
b = np.full(433, 1 / 433)
mk = lambda: sk.PointProblem(inst.x, inst.y, a, b, inst.epsilon)
warm = sk.solve(mk().with_epsilon(inst.basis_eps), tol=1e-10)
basis = sk.top_modes(mk().with_epsilon(inst.basis_eps), warm.f, warm.g, 6)
world = int(sys.argv[1]) if len(sys.argv) > 1 else 8
for label, fn in (("SK", lambda p: sk.solve(p, tol=1e-9)),
                  ("NR", lambda p: sk.solve(p, tol=1e-9, ell=6, basis=basis, init=(warm.f, warm.g)))):
    out = sk.run_emulated_shards(mk, world, fn)
    for r in range(world):
        d = np.abs(out[r].g - out[0].g)
        t0, tr = out[0].trace, out[r].trace
        first = next((i for i in range(min(len(t0), len(tr)))
                      if t0[i].marginal_error != tr[i].marginal_error or t0[i].semi_dual_value != tr[i].semi_dual_value),
                     None)
        print(label, r, out[r].iterations, int((d > 0).sum()), float(d.max()), "first differing record", first,
              flush=True)
out = sk.run_emulated_shards(mk, world, lambda p: (sk.solve(p, tol=1e-9, max_iter=3),
                                                   sk.ctransform_of_f(p, np.linspace(-0.01, 0.01, NN)),
                                                   sk.ctransform_of_g(p, np.linspace(-0.01, 0.01, 433))))
gref = sk.ctransform_of_f(mk(), np.linspace(-0.01, 0.01, NN))
fref = sk.ctransform_of_g(mk(), np.linspace(-0.01, 0.01, 433))
for r in range(world):
    print("rank", r, "g diff vs rank0", float(np.max(np.abs(out[r][1] - out[0][1]))), "vs unsharded",
          float(np.max(np.abs(out[r][1] - gref))), "f diff", float(np.max(np.abs(out[r][2] - out[0][2]))),
          float(np.max(np.abs(out[r][2] - fref))))
out = [o[0] for o in out]
ref = sk.solve(mk(), tol=1e-9, max_iter=3)
for i in range(3):
    print("iter", i + 1, "unsharded", ref.trace[i].marginal_error, ref.trace[i].marginal_error_inf,
          ref.trace[i].semi_dual_value)
    for r in range(world):
        t = out[r].trace[i]
        print("   rank", r, t.marginal_error, t.marginal_error_inf, t.semi_dual_value)
