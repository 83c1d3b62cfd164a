"""Culled vs dense LSE passes: per-pass time, SK iteration, and a solve to tolerance
with identical start (dev tool). Usage: python tools/cull_probe.py [C4|C3] [n]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np

import paper_2506_14780_b200 as sk
from paper_2506_14780_b200 import generators as G

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
n = int(sys.argv[2]) if len(sys.argv) > 2 else None
inst = G.config(name, n=n, m=n)
cells = inst.n * inst.m
pd = sk.PointProblem(inst.x, inst.y, inst.alpha, inst.beta, inst.epsilon, inst.cost_scale)
pc = sk.PointProblem(inst.x, inst.y, inst.alpha, inst.beta, inst.epsilon, inst.cost_scale)
pc.set_culling(60.0)
for label, p in (("dense", pd), ("cull", pc)):
    ms, kpi = sk.bench_iterations(p, 0, None, iters=10, warmup=3)
    print(f"{label:6s} SK iteration (steady state, from f=0 + 3 warm-up): {ms:.3f} ms", flush=True)
res = {}
for label, p in (("dense", pd), ("cull", pc)):
    t0 = time.perf_counter()
    r = sk.solve(p, tol=1e-9, max_iter=100000, trace=False)
    dt = time.perf_counter() - t0
    res[label] = r
    print(f"{label:6s} SK solve: {r.iterations} iterations, conv {r.converged}, {dt*1e3:.1f} ms "
          f"({dt/r.iterations*1e3:.3f} ms/iter)", flush=True)
a, b = res["dense"], res["cull"]
rel = float(np.max(np.abs(a.f - b.f)) / np.max(np.abs(a.f)))
print(f"cull vs dense: same iterations {a.iterations == b.iterations}, rel f diff {rel:.3e}, "
      f"bitwise {np.array_equal(a.f, b.f)}", flush=True)

# SK-NR(ell): iteration time with a random smooth basis, then a solve from the
# eps' = 2 eps warm start with the top_modes basis, dense vs culled
rng = np.random.default_rng(0)
V = np.linalg.qr(rng.standard_normal((inst.n, inst.ell)))[0] * np.sqrt(inst.n)
basis = sk.SpectralBasis(np.asfortranarray(V), np.asfortranarray(V), np.zeros(inst.ell), inst.epsilon)
for label, p in (("dense", pd), ("cull", pc)):
    ms, kpi = sk.bench_iterations(p, inst.ell, basis, iters=5, warmup=2)
    print(f"{label:6s} SK-NR({inst.ell}) iteration: {ms:.3f} ms ({kpi} kernels)", flush=True)
pw = sk.PointProblem(inst.x, inst.y, inst.alpha, inst.beta, 2 * inst.epsilon, inst.cost_scale)
w = sk.solve(pw, tol=1e-9, trace=False)
b = sk.top_modes(pw, w.f, w.g, inst.ell, method="chebyshev", degree=16, max_power_iters=200000)
out = {}
for label, p in (("dense", pd), ("cull", pc)):
    t0 = time.perf_counter()
    r = sk.solve(p, tol=1e-9, ell=inst.ell, basis=b, init=(w.f, w.g), trace=True)
    dt = time.perf_counter() - t0
    out[label] = r
    print(f"{label:6s} SK-NR solve: {r.iterations} iterations, conv {r.converged}, {dt*1e3:.1f} ms, "
          f"accepted {sum(t.newton_accepted for t in r.trace)}", flush=True)
a, c = out["dense"], out["cull"]
print(f"SK-NR cull vs dense: same iterations {a.iterations == c.iterations}, rel f diff "
      f"{float(np.max(np.abs(a.f - c.f)) / np.max(np.abs(a.f))):.3e}, same accepts "
      f"{[t.newton_accepted for t in a.trace] == [t.newton_accepted for t in c.trace]}", flush=True)
