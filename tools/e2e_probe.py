"""Breakdown of the bench's e2e leg (problem upload, solve, download) at C4 (dev tool)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2506_14780_b200 as sk
from paper_2506_14780_b200 import generators as G

inst = G.config("C4")
K = 50
for rep in range(3):
    t0 = time.perf_counter()
    p = sk.PointProblem(inst.x, inst.y, inst.alpha, inst.beta, inst.epsilon)
    t1 = time.perf_counter()
    r = sk.solve(p, tol=1e-300, max_iter=K, trace=False)
    t2 = time.perf_counter()
    r2 = sk.solve(p, tol=1e-300, max_iter=K, trace=False)
    t3 = time.perf_counter()
    print(f"rep {rep}: create {1e3*(t1-t0):.1f} ms, solve {1e3*(t2-t1):.1f} ms, second solve {1e3*(t3-t2):.1f} ms "
          f"-> {2*inst.n*inst.m*K/(t2-t0)/1e9:.0f} GCells/s e2e", flush=True)
    del p
