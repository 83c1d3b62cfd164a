"""C2 (BASELINE configs[1]): n=m=4096 GMM -> uniform square, max-normalised cost,
anneal eps 0.1 -> 0.001 (x0.5, then 0.001), warm=spectral, ell=16, tol 1e-9:
GPU anneal vs the oracle's anneal (solver.cpp:158-222), each side with its own
top_modes basis, in both accept modes (literal = the reference's Q(f') > Q(f);
stable = the same predicate as dQ > 0).
Writes gpurun_out/c2_anneal_parity_r02.json."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np

import oracle_ref as O
import paper_2506_14780_b200 as sk
from paper_2506_14780_b200 import generators as G

inst = G.config("C2")
eps = list(inst.epsilons)
op = O.Instance(inst.alpha, inst.beta, eps[0], x=inst.x, y=inst.y, cost_div=1.0 / inst.cost_scale)
out = {"config": "C2 n=m=4096, eps " + str(eps) + ", warm=spectral, ell=16, tol=1e-9",
       "oracle_threads": O.max_threads(), "modes": {}}
for mode in ("literal", "stable"):
    gp = sk.PointProblem(inst.x, inst.y, inst.alpha, inst.beta, eps[0], inst.cost_scale)
    t0 = time.time()
    sg = sk.anneal(gp, eps, warm="spectral", ell=inst.ell, accept=mode)
    tg = time.time() - t0
    t0 = time.time()
    with O.accept_mode(mode):
        so = O.anneal(op, eps, warm="spectral", ell=inst.ell)
    to = time.time() - t0
    rel_f = [float(np.max(np.abs(a.f - b["f"])) / np.max(np.abs(b["f"]))) for a, b in zip(sg, so)]
    rel_g = [float(np.max(np.abs(a.g - b["g"])) / np.max(np.abs(b["g"]))) for a, b in zip(sg, so)]
    acc_diff = [sum(1 for x, y in zip([t.newton_accepted for t in a.trace], [bool(t[4]) for t in b["trace"]])
                    if x != y) for a, b in zip(sg, so)]
    row = {"gpu_s": tg, "oracle_s": to,
           "iterations_gpu": [s.iterations for s in sg], "iterations_oracle": [s["iterations"] for s in so],
           "identical_iterations": [s.iterations for s in sg] == [s["iterations"] for s in so],
           "converged_gpu": [s.converged for s in sg], "converged_oracle": [s["converged"] for s in so],
           "differing_accepts_per_stage": acc_diff, "rel_f": rel_f, "rel_g": rel_g, "max_rel_f": max(rel_f)}
    out["modes"][mode] = row
    print(mode, json.dumps(row), flush=True)
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
json.dump(out, open(os.path.join(ROOT, "gpurun_out", "c2_anneal_parity_r02.json"), "w"), indent=1)
