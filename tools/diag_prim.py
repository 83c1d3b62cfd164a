import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import oracle_ref as O
import paper_2506_14780_b200 as sk
from paper_2506_14780_b200 import generators as G
cfg = sys.argv[1]; n = int(sys.argv[2]); K = int(sys.argv[3])
inst = G.config(cfg, n=n, m=n)
op = O.Instance(inst.alpha, inst.beta, inst.epsilon, x=inst.x, y=inst.y, cost_div=1.0 / inst.cost_scale)
ro = O.solve(op, tol=1e-300, max_iter=K)
f = ro["f"]
print("f range", f.min(), f.max())
go = O.ctransform_of_f(op, f)
gp = sk.PointProblem(inst.x, inst.y, inst.alpha, inst.beta, inst.epsilon, inst.cost_scale)
g1 = sk.ctransform_of_f(gp, f)
print("fresh handle rel", np.max(np.abs(g1 - go)) / np.max(np.abs(go)), "argmax", np.argmax(np.abs(g1 - go)))
bad = np.where(np.abs(g1 - go) > 1e-9 * np.max(np.abs(go)))[0]
print("bad count", bad.size, bad[:20])
fo = O.ctransform_of_g(op, go)
f1 = sk.ctransform_of_g(gp, go)
print("row transform rel", np.max(np.abs(f1 - fo)) / np.max(np.abs(fo)))
