"""C2 (BASELINE configs[1]): n=m=4096 GMM -> uniform square, max-normalised cost,
anneal eps 0.1 -> 0.001 (x0.5, then 0.001), warm=spectral, ell=16, tol 1e-9:
GPU anneal vs the oracle's anneal (solver.cpp:158-222). Writes gpurun_out/c2_anneal_parity_r01.json."""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import oracle_ref as O
import paper_2506_14780_b200 as sk
from paper_2506_14780_b200 import generators as G

inst = G.config("C2")
eps = list(inst.epsilons)
gp = sk.PointProblem(inst.x, inst.y, inst.alpha, inst.beta, eps[0], inst.cost_scale)
t0 = time.time()
sg = sk.anneal(gp, eps, warm="spectral", ell=inst.ell)
tg = time.time() - t0
print(f"gpu anneal {tg:.2f}s iterations {[s.iterations for s in sg]}", flush=True)
op = O.Instance(inst.alpha, inst.beta, eps[0], x=inst.x, y=inst.y, cost_div=1.0 / inst.cost_scale)
t0 = time.time()
so = O.anneal(op, eps, warm="spectral", ell=inst.ell)
to = time.time() - t0
print(f"oracle anneal {to:.1f}s iterations {[s['iterations'] for s in so]}", flush=True)
rel = [float(np.max(np.abs(a.f - b["f"])) / np.max(np.abs(b["f"]))) for a, b in zip(sg, so)]
out = {"config": "C2 n=m=4096, eps " + str(eps) + ", warm=spectral, ell=16, tol=1e-9",
       "gpu_s": tg, "oracle_s": to, "oracle_threads": O.max_threads(),
       "iterations_gpu": [s.iterations for s in sg], "iterations_oracle": [s["iterations"] for s in so],
       "converged_gpu": [s.converged for s in sg], "converged_oracle": [s["converged"] for s in so],
       "rel_f": rel}
print(json.dumps(out), flush=True)
json.dump(out, open(os.path.join(ROOT, "gpurun_out", "c2_anneal_parity_r01.json"), "w"), indent=1)

# Second comparison: the same stage logic with the oracle's basis handed to the GPU
# solve (isolates the top_modes rounding: ~1e-8 residual-level basis differences).
prev = None
basis_o = None
shared = {"iterations_gpu": [], "iterations_oracle": [], "rel_f": [], "last_gap_gpu": [], "last_gap_oracle": []}
for s, e in enumerate(eps):
    gp.set_epsilon(e)
    if s == 0:
        rg = sk.solve(gp, tol=1e-9)
        ro = O.solve(op.with_epsilon(e), tol=1e-9)
    else:
        if basis_o is None:
            basis_o = O.top_modes(op.with_epsilon(eps[s - 1]), prev["f"], prev["g"], inst.ell)
        sb = sk.SpectralBasis(basis_o["vectors"], basis_o["vectors_sym"], basis_o["rhos"], eps[s - 1])
        rg = sk.solve(gp, tol=1e-9, ell=inst.ell, basis=sb, init=(prev["f"], prev["g"]))
        ro = O.solve(op.with_epsilon(e), tol=1e-9, ell=inst.ell, V=basis_o["vectors"], init=(prev["f"], prev["g"]))
    shared["iterations_gpu"].append(rg.iterations)
    shared["iterations_oracle"].append(ro["iterations"])
    shared["rel_f"].append(float(np.max(np.abs(rg.f - ro["f"])) / np.max(np.abs(ro["f"]))))
    shared["last_gap_gpu"].append([t.marginal_error for t in rg.trace[-2:]])
    shared["last_gap_oracle"].append([t[0] for t in ro["trace"][-2:]])
    prev = ro
out["shared_basis"] = shared
print(json.dumps(shared), flush=True)
json.dump(out, open(os.path.join(ROOT, "gpurun_out", "c2_anneal_parity_r01.json"), "w"), indent=1)
