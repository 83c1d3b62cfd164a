import sys, threading
import numpy as np
sys.path.insert(0, "/root/repo")
import paper_2506_14780_b200 as sk
from paper_2506_14780_b200 import generators as G
NN = 601
inst = G.config("C1", n=NN, m=433)
a = np.full(NN, 1 / NN); b = np.full(433, 1 / 433)
mk = lambda: sk.PointProblem(inst.x, inst.y, a, b, inst.epsilon)
for order in ("fwd", "rev") * 5:
    world = 8
    sk.comm_init_emulated(world)
    probs = []
    for r in range(world):
        p = mk(); sk.shard(p, r, world); probs.append(p)
    out = [None] * world
    def run(r):
        out[r] = sk.solve(probs[r], tol=1e-9, max_iter=3)
    rs = list(range(world)) if order == "fwd" else list(reversed(range(world)))
    th = [threading.Thread(target=run, args=(r,)) for r in rs]
    for t in th: t.start()
    for t in th: t.join()
    sk.comm_destroy()
    print(order, len(set(o.trace[0].semi_dual_value for o in out)), len(set(o.trace[0].marginal_error for o in out)), len(set(o.trace[2].semi_dual_value for o in out)))
