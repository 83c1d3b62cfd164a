"""Throughput of solve_batch vs one-by-one solves on C1-sized problems (dev tool).
Usage: python tools/batch_probe.py [B] [ell]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np

import paper_2506_14780_b200 as sk
from paper_2506_14780_b200 import generators as G

B = int(sys.argv[1]) if len(sys.argv) > 1 else 32
ell = int(sys.argv[2]) if len(sys.argv) > 2 else 0
probs, bases, inits = [], [], []
for s in range(B):
    inst = G.config("C1", seed=1 + s)
    p = sk.PointProblem(inst.x, inst.y, inst.alpha, inst.beta, inst.epsilon)
    probs.append(p)
    if ell:
        warm = sk.solve(p.with_epsilon(inst.basis_eps))
        bases.append(sk.top_modes(p.with_epsilon(inst.basis_eps), warm.f, warm.g, ell))
        inits.append((warm.f, warm.g))
kw = dict(tol=1e-9, ell=ell, bases=bases or None, inits=inits or None)
sk.solve_batch(probs[:2], **dict(kw, bases=bases[:2] or None, inits=inits[:2] or None))  # warm-up
t0 = time.perf_counter()
res = sk.solve_batch(probs, **kw)
tb = time.perf_counter() - t0
t0 = time.perf_counter()
one = [sk.solve(p, tol=1e-9, ell=ell, basis=bases[i] if ell else None, init=inits[i] if ell else None,
                trace=False) for i, p in enumerate(probs)]
ts = time.perf_counter() - t0
same = all(np.array_equal(a.f, b.f) and a.iterations == b.iterations for a, b in zip(res, one))
its = [r.iterations for r in res]
print(f"B={B} ell={ell}: batch {tb*1e3:.1f} ms ({B/tb:.1f} solves/s), one-by-one {ts*1e3:.1f} ms "
      f"({B/ts:.1f} solves/s), speed-up {ts/tb:.2f}x, iterations {min(its)}..{max(its)}, bitwise-equal {same}")
