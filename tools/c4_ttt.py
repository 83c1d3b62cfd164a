"""C4 time-to-tolerance on one B200: plain SK vs SK-NR(32) with eps'=2 eps warm
start and a Chebyshev-filtered basis. Writes gpurun_out/c4_ttt_r01.json
(c4_ttt_cull_r01.json with --cull: opt-in culled LSE passes on every problem)."""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2506_14780_b200 as sk
from paper_2506_14780_b200 import generators as G
cull = "--cull" in sys.argv
lanczos = "--lanczos" in sys.argv
sys.argv = [a for a in sys.argv if a not in ("--cull", "--lanczos")]
c = G.config("C4")
out = {"config": "C4 n=m=65536 d=2 eps=5e-4 tol=1e-9", "ell": c.ell, "warm_eps": c.basis_eps}
p = sk.PointProblem(c.x, c.y, c.alpha, c.beta, c.epsilon)
if cull:
    p.set_culling(60.0)
t0 = time.perf_counter()
r = sk.solve(p, tol=1e-9, max_iter=int(sys.argv[1]) if len(sys.argv) > 1 else 200000, trace=False)
out["sk"] = {"iterations": r.iterations, "converged": r.converged, "s": time.perf_counter() - t0}
print(out["sk"], flush=True)
pw = sk.PointProblem(c.x, c.y, c.alpha, c.beta, c.basis_eps)
if cull:
    pw.set_culling(60.0)
t0 = time.perf_counter()
w = sk.solve(pw, tol=1e-9, trace=False)
tw = time.perf_counter() - t0
t0 = time.perf_counter()
b = sk.top_modes(pw, w.f, w.g, c.ell, method="lanczos" if lanczos else "chebyshev", degree=12 if lanczos else 16,
                 max_power_iters=200000)
tb = time.perf_counter() - t0
print("basis", b.sweeps, tb, b.rhos[:4], flush=True)
t0 = time.perf_counter()
r2 = sk.solve(p, tol=1e-9, ell=c.ell, basis=b, init=(w.f, w.g), trace=True)
tn = time.perf_counter() - t0
out["sknr"] = {"iterations": r2.iterations, "converged": r2.converged, "main_s": tn, "warm_iterations": w.iterations,
               "warm_s": tw, "basis_method": "lanczos(12)" if lanczos else "chebyshev(16)", "basis_applications": b.sweeps, "basis_s": tb,
               "end_to_end_s": tw + tb + tn, "accepted": sum(t.newton_accepted for t in r2.trace)}
print(out["sknr"], flush=True)
out["culling"] = cull
json.dump(out, open(os.path.join(ROOT, "gpurun_out", ("c4_ttt_cull" if cull else "c4_ttt") +
                                  ("_lanczos" if lanczos else "") + "_r01.json"), "w"), indent=1)
