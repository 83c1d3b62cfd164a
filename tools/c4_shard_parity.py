"""C4 parity across R on one GPU: the row-sharded path with R emulated ranks
(sknr_comm_init_emulated) against the unsharded solve -- SK to tolerance and
SK-NR(32) from the eps' warm start. Writes gpurun_out/c4_shard_parity_r01.json."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np

import paper_2506_14780_b200 as sk
from paper_2506_14780_b200 import generators as G

R = int(sys.argv[1]) if len(sys.argv) > 1 else 8
c = G.config("C4")
mk = lambda: sk.PointProblem(c.x, c.y, c.alpha, c.beta, c.epsilon)
rel = lambda a, b: float(np.max(np.abs(a - b)) / np.max(np.abs(b)))
out = {"config": "C4 n=m=65536 d=2 eps=5e-4 tol=1e-9", "R": R}
t0 = time.perf_counter()
ref = sk.solve(mk(), tol=1e-9, trace=False)
out["sk_unsharded"] = {"iterations": ref.iterations, "s": time.perf_counter() - t0}
t0 = time.perf_counter()
res = sk.run_emulated_shards(mk, R, lambda p: sk.solve(p, tol=1e-9, trace=False))
out["sk_sharded"] = {"iterations": [r.iterations for r in res], "s": time.perf_counter() - t0,
                     "rel_f": rel(res[0].f, ref.f), "rel_g": rel(res[0].g, ref.g),
                     "ranks_identical": all(np.array_equal(r.g, res[0].g) for r in res)}
print(out, flush=True)
pw = sk.PointProblem(c.x, c.y, c.alpha, c.beta, c.basis_eps)
w = sk.solve(pw, tol=1e-9, trace=False)
b = sk.top_modes(pw, w.f, w.g, c.ell, method="chebyshev", degree=16, max_power_iters=200000)
ref2 = sk.solve(mk(), tol=1e-9, ell=c.ell, basis=b, init=(w.f, w.g))
res2 = sk.run_emulated_shards(mk, R, lambda p: sk.solve(p, tol=1e-9, ell=c.ell, basis=b, init=(w.f, w.g)))
out["sknr_unsharded"] = {"iterations": ref2.iterations, "accepted": sum(t.newton_accepted for t in ref2.trace)}
out["sknr_sharded"] = {"iterations": [r.iterations for r in res2],
                       "accepted": [sum(t.newton_accepted for t in r.trace) for r in res2][:1],
                       "rel_f": rel(res2[0].f, ref2.f), "rel_g": rel(res2[0].g, ref2.g),
                       "same_accepts": [t.newton_accepted for t in res2[0].trace] ==
                                       [t.newton_accepted for t in ref2.trace],
                       "ranks_identical": all(np.array_equal(r.g, res2[0].g) for r in res2)}
print(out, flush=True)
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
json.dump(out, open(os.path.join(ROOT, "gpurun_out", "c4_shard_parity_r01.json"), "w"), indent=1)
