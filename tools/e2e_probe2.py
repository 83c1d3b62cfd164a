"""Which phase of the bench's repeated e2e runs is slow (dev tool)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2506_14780_b200 as sk
from paper_2506_14780_b200 import generators as G

inst = G.config("C4")
K = 50
prob = sk.PointProblem(inst.x, inst.y, inst.alpha, inst.beta, inst.epsilon)
sk.bench_iterations(prob, 0, None, iters=10, warmup=3, flush_l2=True)
res = None
for rep in range(5):
    t0 = time.perf_counter()
    p = sk.PointProblem(inst.x, inst.y, inst.alpha, inst.beta, inst.epsilon)
    t1 = time.perf_counter()
    r = sk.solve(p, tol=1e-300, max_iter=K, trace=False)
    t2 = time.perf_counter()
    res = r
    t3 = time.perf_counter()
    print(f"rep {rep}: create {1e3*(t1-t0):.1f} ms, solve {1e3*(t2-t1):.1f} ms, rebind {1e3*(t3-t2):.1f} ms", flush=True)
    del p
