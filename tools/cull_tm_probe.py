"""top_modes with and without culled operator passes (dev tool)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np

import paper_2506_14780_b200 as sk
from paper_2506_14780_b200 import generators as G

n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
c = G.config("C4", n=n, m=n)
pw = sk.PointProblem(c.x, c.y, c.alpha, c.beta, c.basis_eps)
w = sk.solve(pw, tol=1e-9, trace=False)
for cull in (0.0, 60.0):
    pw.set_culling(cull)
    k0 = sk.kernel_launch_count()
    d0 = sk.debug_counters(pw)
    t0 = time.perf_counter()
    b = sk.top_modes(pw, w.f, w.g, c.ell, method="chebyshev", degree=16, max_power_iters=200000)
    dt = time.perf_counter() - t0
    print(f"cull={cull}: {dt*1e3:.1f} ms, {b.sweeps} applications, launches {sk.kernel_launch_count()-k0}, "
          f"rho[:3] {b.rhos[:3]}", flush=True)
    d1 = sk.debug_counters(pw)
    tested, kept = d1["cull_tested"] - d0["cull_tested"], d1["cull_kept"] - d0["cull_kept"]
    print(f"  cull groups tested {tested}, kept {kept} ({kept / max(tested, 1):.3f})", flush=True)
    for which in (4,):
        ms, kms = sk.bench_pass(pw, which, c.ell, passes=3)
        print(f"  bench_pass {which}: {ms:.3f} ms (kernel {kms:.3f})", flush=True)
