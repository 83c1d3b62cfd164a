"""Partial-trajectory parity (K SK iterations from f = 0, then K_NR SK-NR
iterations with a smooth basis) for C3 and C5 (stored and on-the-fly cost).
Writes gpurun_out/partial_parity_r01.json."""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import oracle_ref as O
import paper_2506_14780_b200 as sk
from paper_2506_14780_b200 import generators as G

def rel(a, b):
    return float(np.max(np.abs(a - b)) / np.max(np.abs(b)))

def smooth_basis(x, alpha, ell):
    rng = np.random.default_rng(0)
    proj = rng.standard_normal((x.shape[1], 2))
    z = x @ proj
    z = (z - z.min(0)) / (z.max(0) - z.min(0))
    cols = []
    for a in range(8):
        for b in range(8):
            if a == 0 and b == 0:
                continue
            cols.append(np.cos(np.pi * a * z[:, 0]) * np.cos(np.pi * b * z[:, 1]))
    V = np.stack(cols[:ell], 1)
    w = np.sqrt(alpha)[:, None]
    Vs = V * w
    Vs -= np.sqrt(alpha)[:, None] * (np.sqrt(alpha) @ Vs)[None, :]
    Q, _ = np.linalg.qr(Vs)
    return np.asfortranarray(Q / w)

out = {}
cases = [("C3", "auto", 10, 3), ("C5", "stored", 4, 2), ("C5", "onthefly", 4, 2)]
for name, mode, K, KN in cases:
    c = G.config(name)
    gp = sk.PointProblem(c.x, c.y, c.alpha, c.beta, c.epsilon, c.cost_scale, cost_mode=mode)
    op = O.Instance(c.alpha, c.beta, c.epsilon, x=c.x, y=c.y, cost_div=1.0 / c.cost_scale)
    t0 = time.time(); rg = sk.solve(gp, tol=1e-300, max_iter=K); tg = time.time() - t0
    t0 = time.time(); ro = O.solve(op, tol=1e-300, max_iter=K); to = time.time() - t0
    V = smooth_basis(c.x, c.alpha, c.ell)
    bas = sk.SpectralBasis(V, V, np.zeros(c.ell), c.epsilon)
    init = (ro["f"], ro["g"])
    t0 = time.time(); ng = sk.solve(gp, tol=1e-300, max_iter=KN, ell=c.ell, basis=bas, init=init); tg2 = time.time() - t0
    t0 = time.time(); no = O.solve(op, tol=1e-300, max_iter=KN, ell=c.ell, V=V, init=init); to2 = time.time() - t0
    key = f"{name}_{mode}"
    out[key] = {"n": c.n, "m": c.m, "d": c.x.shape[1], "eps": c.epsilon, "cost_path": gp.cost_path,
                "sk": {"iterations": K, "gpu_s": tg, "oracle_s": to, "rel_f": rel(rg.f, ro["f"]), "rel_g": rel(rg.g, ro["g"]),
                       "max_rel_gap_diff": max(abs(a.marginal_error - b[0]) / b[0] for a, b in zip(rg.trace, ro["trace"]))},
                "sknr": {"ell": c.ell, "iterations": KN, "gpu_s": tg2, "oracle_s": to2, "rel_f": rel(ng.f, no["f"]),
                         "accepted_gpu": [bool(t.newton_accepted) for t in ng.trace],
                         "accepted_oracle": [bool(t[4]) for t in no["trace"]],
                         "max_abs_Q_diff": max(abs(a.semi_dual_value - b[2]) for a, b in zip(ng.trace, no["trace"]))}}
    print(key, json.dumps(out[key]), flush=True)
    del gp
json.dump(out, open(os.path.join(ROOT, "gpurun_out", "partial_parity_r01.json"), "w"), indent=1)
