import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import oracle_ref as O
import paper_2506_14780_b200 as sk
from paper_2506_14780_b200 import generators as G
cfg = sys.argv[1]; n = int(sys.argv[2])
inst = G.config(cfg, n=n, m=n)
op = O.Instance(inst.alpha, inst.beta, inst.epsilon, x=inst.x, y=inst.y, cost_div=1.0 / inst.cost_scale)
ro = O.solve(op, tol=1e-300, max_iter=3)
f = ro["f"]
go = O.ctransform_of_f(op, f)
gp = sk.PointProblem(inst.x, inst.y, inst.alpha, inst.beta, inst.epsilon, inst.cost_scale)
def chk(tag):
    g1 = sk.ctransform_of_f(gp, f)
    print(f"{tag:30s} rel {np.max(np.abs(g1 - go)) / np.max(np.abs(go)):.3e}", flush=True)
chk("fresh")
chk("fresh again")
sk.solve(gp, tol=1e-300, max_iter=3)
chk("after solve(3)")
chk("again")
sk.solve(gp, tol=1e-300, max_iter=3, trace=False)
chk("after solve notrace")
gp.set_epsilon(inst.epsilon)
chk("after set_epsilon")
g2 = sk.ctransform_of_g(gp, go)
chk("after ctransform_of_g")
