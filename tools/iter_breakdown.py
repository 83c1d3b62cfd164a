"""Per-iteration overhead study (dev tool): SK iteration time for a config vs the
sum of its kernels' durations (run the same command under ncu's launch list to
get the latter). Usage: python tools/iter_breakdown.py C3 [iters]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2506_14780_b200 as sk
from paper_2506_14780_b200 import generators as G

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 20
inst = G.config(name)
p = sk.PointProblem(inst.x, inst.y, inst.alpha, inst.beta, inst.epsilon, inst.cost_scale)
ms, kpi = sk.bench_iterations(p, 0, None, iters=iters, warmup=3)
print(f"{name} n={inst.n} m={inst.m} d={inst.x.shape[1]}: SK iteration {ms:.4f} ms, {kpi} kernels", flush=True)
if len(sys.argv) > 3 and sys.argv[3] == "nr":
    import numpy as np
    rng = np.random.default_rng(0)
    V = np.linalg.qr(rng.standard_normal((inst.n, inst.ell)))[0] * np.sqrt(inst.n)
    basis = sk.SpectralBasis(np.asfortranarray(V), np.asfortranarray(V), np.zeros(inst.ell), inst.epsilon)
    ms, kpi = sk.bench_iterations(p, inst.ell, basis, iters=iters, warmup=3)
    print(f"{name}: SK-NR({inst.ell}) iteration {ms:.4f} ms, {kpi} kernels", flush=True)
