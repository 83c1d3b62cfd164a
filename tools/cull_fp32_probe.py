import sys, os, time, json
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2506_14780_b200 as sk
from paper_2506_14780_b200 import generators as G
c = G.config("C4")
out = {}
for prec in (64, 32):
    p = sk.PointProblem(c.x, c.y, c.alpha, c.beta, c.epsilon); p.set_culling(60.0); p.set_precision(prec)
    ms, kpi = sk.bench_iterations(p, 0, None, iters=20, warmup=3, flush_l2=True)
    out[f"cull_sk_iter_ms_{prec}"] = ms
    print(prec, ms, flush=True)
rel = lambda a, b: float(np.max(np.abs(a - b)) / np.max(np.abs(b)))
res = {}
for prec in (64, 32):
    pw = sk.PointProblem(c.x, c.y, c.alpha, c.beta, c.basis_eps); pw.set_culling(60.0); pw.set_precision(prec)
    t0 = time.perf_counter(); w = sk.solve(pw, tol=1e-9, trace=False); tw = time.perf_counter() - t0
    pw.set_precision(64)
    t0 = time.perf_counter(); b = sk.top_modes(pw, w.f, w.g, c.ell, method="lanczos", degree=12, max_power_iters=200000); tb = time.perf_counter() - t0
    pm = sk.PointProblem(c.x, c.y, c.alpha, c.beta, c.epsilon); pm.set_culling(60.0)
    t0 = time.perf_counter(); r = sk.solve(pm, tol=1e-9, ell=c.ell, basis=b, init=(w.f, w.g), trace=False); tm = time.perf_counter() - t0
    res[prec] = r
    out[f"sknr_e2e_cull_warm{prec}"] = {"warm_it": w.iterations, "warm_s": tw, "basis_s": tb, "basis_apps": b.sweeps,
                                        "main_it": r.iterations, "main_s": tm, "total_s": tw + tb + tm}
    print(prec, out[f"sknr_e2e_cull_warm{prec}"], flush=True)
out["rel_f_32_vs_64"] = rel(res[32].f, res[64].f)
print(json.dumps(out), flush=True)
