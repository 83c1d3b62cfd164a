"""Quick device timing of the individual passes at a BASELINE config (dev tool)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np

import paper_2506_14780_b200 as sk
from paper_2506_14780_b200 import generators as G

cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
n = int(sys.argv[2]) if len(sys.argv) > 2 else None
t0 = time.time()
inst = G.config(cfg, n=n, m=n)
print(f"{cfg}: n={inst.n} m={inst.m} d={inst.x.shape[1]} gen {time.time()-t0:.1f}s", flush=True)
p = sk.PointProblem(inst.x, inst.y, inst.alpha, inst.beta, inst.epsilon, inst.cost_scale)
cells = inst.n * inst.m
names = {0: "col LSE (full)", 1: "row LSE (full)", 2: "col sum kernel", 3: f"block pass ell={inst.ell}"}
for which in (0, 1, 2, 3):
    ms, kms = sk.bench_pass(p, which, inst.ell, passes=5)
    print(f"{names[which]:24s} pass {ms:8.3f} ms  kernel {kms:8.3f} ms  "
          f"{cells/ms/1e6:8.1f} GCells/s (pass)  {cells/kms/1e6:8.1f} GCells/s (kernel)", flush=True)
ms, kpi = sk.bench_iterations(p, 0, None, iters=5)
print(f"SK iteration      {ms:8.3f} ms  kernels/iter {kpi}", flush=True)
rng = np.random.default_rng(0)
V = np.linalg.qr(rng.standard_normal((inst.n, inst.ell)))[0] * np.sqrt(inst.n)
basis = sk.SpectralBasis(np.asfortranarray(V), np.asfortranarray(V), np.zeros(inst.ell), inst.epsilon)
ms, kpi = sk.bench_iterations(p, inst.ell, basis, iters=3)
print(f"SK-NR iteration   {ms:8.3f} ms  kernels/iter {kpi}", flush=True)
