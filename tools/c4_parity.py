"""C4 (n=m=65536, d=2, eps=5e-4) parity of the GPU solver against the CPU oracle
over K iterations from the same initial potentials (the oracle cannot reach
tolerance at this size: ~13 s per SK iteration on 16 cores). SK from f=0, then
SK-NR(32) from the SK iterate with a smooth L2(alpha)-orthonormal basis.
Writes profiles/c4_parity_r01.json."""
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

K_SK = int(sys.argv[1]) if len(sys.argv) > 1 else 8
K_NR = int(sys.argv[2]) if len(sys.argv) > 2 else 4
inst = G.config("C4")
n, m, ell = inst.n, inst.m, inst.ell
gp = sk.PointProblem(inst.x, inst.y, inst.alpha, inst.beta, inst.epsilon)
op = O.Instance(inst.alpha, inst.beta, inst.epsilon, x=inst.x, y=inst.y)
print("oracle threads", O.max_threads(), flush=True)

def rel(a, b):
    return float(np.max(np.abs(a - b)) / np.max(np.abs(b)))

out = {"config": "C4 n=m=65536 d=2 eps=5e-4", "oracle_threads": O.max_threads()}
t0 = time.time()
rg = sk.solve(gp, tol=1e-300, max_iter=K_SK)
tg = time.time() - t0
t0 = time.time()
ro = O.solve(op, tol=1e-300, max_iter=K_SK)
to = time.time() - t0
out["sk"] = {"iterations": K_SK, "gpu_s": tg, "oracle_s": to, "rel_f": rel(rg.f, ro["f"]), "rel_g": rel(rg.g, ro["g"]),
             "marginal_error_gpu": [t.marginal_error for t in rg.trace],
             "marginal_error_oracle": [t[0] for t in ro["trace"]],
             "max_rel_marginal_error_diff": max(abs(a.marginal_error - b[0]) / b[0] for a, b in zip(rg.trace, ro["trace"]))}
print(json.dumps(out["sk"])[:400], flush=True)

# smooth basis: products of cosines in x, alpha-mean-zero, L2(alpha)-orthonormal
x = inst.x
cols = []
for a in range(0, 8):
    for b in range(0, 8):
        if a == 0 and b == 0:
            continue
        cols.append(np.cos(np.pi * a * x[:, 0]) * np.cos(np.pi * b * x[:, 1]))
        if len(cols) == ell:
            break
    if len(cols) == ell:
        break
V = np.stack(cols, 1)
w = np.sqrt(inst.alpha)[:, None]
Vs = V * w
Vs -= np.sqrt(inst.alpha)[:, None] * (np.sqrt(inst.alpha) @ Vs)[None, :]
Q, _ = np.linalg.qr(Vs)
Vb = np.asfortranarray(Q / w)
basis = sk.SpectralBasis(Vb, np.asfortranarray(Q), np.zeros(ell), inst.epsilon)
init = (ro["f"], ro["g"])
t0 = time.time()
ng = sk.solve(gp, tol=1e-300, max_iter=K_NR, ell=ell, basis=basis, init=init)
tg = time.time() - t0
t0 = time.time()
no = O.solve(op, tol=1e-300, max_iter=K_NR, ell=ell, V=Vb, init=init)
to = time.time() - t0
out["sknr"] = {"ell": ell, "iterations": K_NR, "gpu_s": tg, "oracle_s": to, "rel_f": rel(ng.f, no["f"]),
               "rel_g": rel(ng.g, no["g"]),
               "accepted_gpu": [bool(t.newton_accepted) for t in ng.trace],
               "accepted_oracle": [bool(t[4]) for t in no["trace"]],
               "Q_gpu": [t.semi_dual_value for t in ng.trace], "Q_oracle": [t[2] for t in no["trace"]],
               "marginal_error_gpu": [t.marginal_error for t in ng.trace],
               "marginal_error_oracle": [t[0] for t in no["trace"]]}
print(json.dumps(out["sknr"])[:600], flush=True)
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
json.dump(out, open(os.path.join(ROOT, "gpurun_out", "c4_parity_r01.json"), "w"), indent=1)
