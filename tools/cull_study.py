"""How many cells of a C4-like LSE pass are negligible (E_ij - L_j < -T) and how many
Morton-ordered box pairs could be skipped (dev study)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np

import paper_2506_14780_b200 as sk
from paper_2506_14780_b200 import generators as G

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
name = sys.argv[2] if len(sys.argv) > 2 else "C4"
inst = G.config(name, n=n, m=n)
eps = inst.epsilon
p = sk.PointProblem(inst.x, inst.y, inst.alpha, inst.beta, eps, inst.cost_scale)
for it in (20, 200, 100000):
    r = sk.solve(p, tol=1e-9, max_iter=it, trace=False)
    f = r.f
    x, y = inst.x, inst.y
    d = x.shape[1]

    def morton(pts):
        lo, hi = pts.min(0), pts.max(0)
        q = np.clip(((pts - lo) / (hi - lo + 1e-12) * 1023).astype(np.int64), 0, 1023)
        code = np.zeros(len(pts), dtype=np.int64)
        for b in range(10):
            for k in range(d):
                code |= ((q[:, k] >> b) & 1) << (d * b + k)
        return np.argsort(code, kind="stable")

    pi, pj = morton(x), morton(y)
    xs, ys, fs, las = x[pi], y[pj], f[pi], np.log(inst.alpha[pi])
    res = {}
    for T in (40, 60):
        keep = 0
        boxes = {}
        for j0 in range(0, n, 1024):
            C = ((xs[:, None, :] - ys[None, j0:j0 + 1024, :]) ** 2).sum(-1) * inst.cost_scale
            E = las[:, None] + (fs[:, None] - C) / eps
            L = np.log(np.exp(E - E.max(0)).sum(0)) + E.max(0)
            rel = E - L[None, :]
            keep += (rel > -T).sum()
            for ci, cj in ((256, 256), (64, 256), (32, 32)):
                blk = rel.reshape(n // ci, ci, 1024 // cj, cj).max(axis=(1, 3))
                boxes[(ci, cj)] = boxes.get((ci, cj), 0) + (blk > -T).sum()
        res[T] = (keep / n / n, {k: v / ((n // k[0]) * (n // k[1])) for k, v in boxes.items()})
    print(f"{name} n={n} after {r.iterations} SK iterations (err tol 1e-9 conv={r.converged}):", flush=True)
    for T, (c, b) in res.items():
        print(f"  T={T}: cells kept {c:.3f}; box pairs kept " +
              ", ".join(f"{k[0]}x{k[1]}: {v:.3f}" for k, v in b.items()), flush=True)
