import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import paper_2506_14780_b200 as sk
from paper_2506_14780_b200 import generators as G
cfg = sys.argv[1]; K = int(sys.argv[2])
inst = G.config(cfg)
gp = sk.PointProblem(inst.x, inst.y, inst.alpha, inst.beta, inst.epsilon, inst.cost_scale)
t0 = time.time()
r = sk.solve(gp, tol=1e-9, max_iter=K)
print(f"iters {r.iterations} conv {r.converged} {time.time()-t0:.1f}s", sk.debug_counters(gp))
errs = [t.marginal_error for t in r.trace]
for k in list(range(0, len(errs), max(1, len(errs)//40))) + [len(errs)-1]:
    print(k + 1, f"{errs[k]:.6e}  Q {r.trace[k].semi_dual_value:.15e}")
print("f finite", np.all(np.isfinite(r.f)), "range", r.f.min(), r.f.max())
