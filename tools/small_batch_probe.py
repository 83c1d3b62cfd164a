"""Throughput: solve_small_batch (one CTA per problem) vs solve_batch vs one-by-one (dev tool)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np

import paper_2506_14780_b200 as sk
from paper_2506_14780_b200 import generators as G

B = int(sys.argv[1]) if len(sys.argv) > 1 else 148
insts = [G.config("C1", seed=1 + s) for s in range(B)]
tup = [(c.x, c.y, c.alpha, c.beta, c.epsilon) for c in insts]
sk.solve_small_batch(tup[:2], tol=1e-9)
t0 = time.perf_counter()
rs = sk.solve_small_batch(tup, tol=1e-9)
t_small = time.perf_counter() - t0
probs = [sk.PointProblem(*t) for t in tup[:32]]
sk.solve_batch(probs[:2], tol=1e-9)
t0 = time.perf_counter()
rb = sk.solve_batch(probs, tol=1e-9)
t_graph = (time.perf_counter() - t0) * B / 32
one = sk.solve(probs[0], tol=1e-9, trace=False)
same = all(a.iterations == b.iterations for a, b in zip(rs[:32], rb))
print(f"B={B}: small-batch kernel {t_small*1e3:.1f} ms ({B/t_small:.0f} solves/s); graph batch (scaled from 32) "
      f"{t_graph*1e3:.1f} ms ({B/t_graph:.0f} solves/s); iterations equal to solve_batch: {same}; "
      f"max rel f diff {max(float(np.max(np.abs(a.f-b.f))/np.max(np.abs(b.f))) for a, b in zip(rs[:32], rb)):.2e}",
      flush=True)

# single-problem latency: a CTA group per problem (G = 32 at C1, up to one CTA per SM at C2)
for name, eps in (("C1", None), ("C2", 0.02), ("C2", 1e-3)):
    c = G.config(name)
    e = c.epsilon if eps is None else eps
    tup1 = (c.x, c.y, c.alpha, c.beta, e, c.cost_scale)
    sk.solve_small_batch([tup1], tol=1e-9)
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        r1 = sk.solve_small_batch([tup1], tol=1e-9)[0]
        ts.append(time.perf_counter() - t0)
    p1 = sk.PointProblem(c.x, c.y, c.alpha, c.beta, e, c.cost_scale)
    sk.solve(p1, tol=1e-9, trace=False)
    tg = []
    for _ in range(3):
        t0 = time.perf_counter()
        rg = sk.solve(p1, tol=1e-9, trace=False)
        tg.append(time.perf_counter() - t0)
    print(f"{name} eps={e}: group kernel {min(ts)*1e3:.2f} ms ({r1.iterations} it, "
          f"{min(ts)/r1.iterations*1e6:.1f} us/it) vs graph solve {min(tg)*1e3:.2f} ms ({rg.iterations} it); "
          f"rel f diff {float(np.max(np.abs(r1.f-rg.f))/np.max(np.abs(rg.f))):.2e}", flush=True)
