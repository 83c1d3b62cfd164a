"""top_modes: subspace vs Chebyshev vs block Lanczos (applications, time, agreement)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np

import paper_2506_14780_b200 as sk
from paper_2506_14780_b200 import generators as G

name = sys.argv[1] if len(sys.argv) > 1 else "C1"
n = int(sys.argv[2]) if len(sys.argv) > 2 else None
c = G.config(name, n=n, m=n)
pw = sk.PointProblem(c.x, c.y, c.alpha, c.beta, c.basis_eps or 2 * c.epsilon, c.cost_scale)
w = sk.solve(pw, tol=1e-9, trace=False)
res = {}
for method, deg in (("subspace", 1), ("chebyshev", 16), ("lanczos", 8), ("lanczos", 12)):
    if method == "subspace" and c.n > 20000:
        continue
    t0 = time.perf_counter()
    try:
        b = sk.top_modes(pw, w.f, w.g, c.ell, method=method, degree=deg, max_power_iters=600 if method == "lanczos" else 200000)
    except Exception as e:  # noqa: BLE001
        print(method, deg, "failed:", e, flush=True)
        continue
    dt = time.perf_counter() - t0
    res[(method, deg)] = b
    print(f"{name} {method}({deg}): {b.sweeps} applications, {dt*1e3:.1f} ms, rho[:3] {b.rhos[:3]}", flush=True)
ref = res.get(("chebyshev", 16))
for k, b in res.items():
    if ref is not None:
        print(k, "rho rel diff", float(np.max(np.abs(b.rhos - ref.rhos) / np.abs(ref.rhos))),
              "projector distance", sk.projector_distance(b, ref), flush=True)
