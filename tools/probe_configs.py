"""Dev probe: pass timings for C3/C5 and time-to-tolerance for a config."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np

import paper_2506_14780_b200 as sk
from paper_2506_14780_b200 import generators as G

what = sys.argv[1]
if what == "passes":
    for cfg in sys.argv[2:]:
        t0 = time.time()
        inst = G.config(cfg)
        print(f"{cfg}: n={inst.n} m={inst.m} d={inst.x.shape[1]} gen {time.time()-t0:.1f}s", flush=True)
        p = sk.PointProblem(inst.x, inst.y, inst.alpha, inst.beta, inst.epsilon, inst.cost_scale)
        cells = inst.n * inst.m
        for which in (0, 1, 3):
            ms, kms = sk.bench_pass(p, which, inst.ell, passes=5)
            print(f"  which={which} pass {ms:8.3f} ms kernel {kms:8.3f} ms {cells/kms/1e6:8.1f} GCells/s",
                  flush=True)
        del p
elif what == "c5":
    inst = G.config("C5")
    cells = inst.n * inst.m
    for mode in ("stored", "onthefly"):
        p = sk.PointProblem(inst.x, inst.y, inst.alpha, inst.beta, inst.epsilon, inst.cost_scale, cost_mode=mode)
        for which in (0, 1, 3):
            ms, kms = sk.bench_pass(p, which, inst.ell, passes=5)
            print(f"C5 {mode:9s} ({p.cost_path}) which={which} pass {ms:8.3f} ms kernel {kms:8.3f} ms "
                  f"{cells/kms/1e6:8.1f} GCells/s", flush=True)
        del p
elif what == "ttt":
    cfg = sys.argv[2]
    inst = G.config(cfg)
    p = sk.PointProblem(inst.x, inst.y, inst.alpha, inst.beta, inst.epsilon, inst.cost_scale)
    t0 = time.time()
    r = sk.solve(p, tol=1e-9, max_iter=int(sys.argv[3]) if len(sys.argv) > 3 else 100000, trace=True)
    t1 = time.time()
    print(f"{cfg} SK: iters={r.iterations} conv={r.converged} {t1-t0:.2f}s  last err "
          f"{r.trace[-1].marginal_error:.3e}", flush=True)
    if inst.basis_eps:
        pw = sk.PointProblem(inst.x, inst.y, inst.alpha, inst.beta, inst.basis_eps, inst.cost_scale)
        t0 = time.time()
        w = sk.solve(pw, tol=1e-9, trace=False)
        t1 = time.time()
        print(f"  warm eps'={inst.basis_eps}: iters={w.iterations} {t1-t0:.2f}s", flush=True)
        b = sk.top_modes(pw, w.f, w.g, inst.ell)
        t2 = time.time()
        print(f"  top_modes ell={inst.ell}: sweeps={b.sweeps} {t2-t1:.2f}s rhos[:4]={b.rhos[:4]}", flush=True)
        r2 = sk.solve(p, tol=1e-9, ell=inst.ell, basis=b, init=(w.f, w.g), trace=True)
        t3 = time.time()
        print(f"  SK-NR: iters={r2.iterations} conv={r2.converged} {t3-t2:.2f}s accepted="
              f"{sum(t.newton_accepted for t in r2.trace)}", flush=True)
