"""Seed sweep of the Newton accept test, literal vs stable, GPU vs oracle.

For C1-shaped problems (n = m = 512, eps = 1e-2, ell = 10, eps' = 2e-2 warm start and
basis from the oracle, shared by both sides) and seeds 1..S, run the SK-NR main solve on
the GPU and on the oracle in both accept modes and count: iterations, iterations where
the two sides' decisions differ, and those differences above the step noise floor
(the oracle's step max|f'-f| > 1e-10 max|f|). Writes gpurun_out/accept_modes_r02.json (copied to profiles/ by hand).

  python tools/accept_modes.py [S]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np

import oracle_ref as O
import paper_2506_14780_b200 as sk
from paper_2506_14780_b200 import generators as G


def main(S):
    rows = []
    for seed in range(1, S + 1):
        c = G.config("C1", seed=seed)
        gp = sk.PointProblem(c.x, c.y, c.alpha, c.beta, c.epsilon)
        op = O.Instance(c.alpha, c.beta, c.epsilon, x=c.x, y=c.y)
        w = O.solve(op.with_epsilon(c.basis_eps), tol=1e-9, trace=False)
        b = O.top_modes(op.with_epsilon(c.basis_eps), w["f"], w["g"], c.ell)
        sb = sk.SpectralBasis(b["vectors"], b["vectors_sym"], b["rhos"], c.basis_eps)
        row = {"seed": seed}
        for mode in ("literal", "stable"):
            rg = sk.solve(gp, tol=1e-9, ell=c.ell, basis=sb, init=(w["f"], w["g"]), accept=mode)
            with O.accept_mode(mode):
                ro = O.solve(op, tol=1e-9, ell=c.ell, V=b["vectors"], init=(w["f"], w["g"]))
            fs = float(np.max(np.abs(ro["f"])))
            diff = [k + 1 for k, (tg, to) in enumerate(zip(rg.trace, ro["trace"]))
                    if tg.newton_accepted != bool(to[4])]
            sig = [k for k in diff if ro["trace"][k - 1][6] > 1e-10 * fs]
            row[mode] = {"iterations_gpu": rg.iterations, "iterations_oracle": ro["iterations"],
                         "attempts": sum(1 for t in ro["trace"] if t[3]),
                         "accepts_gpu": sum(t.newton_accepted for t in rg.trace),
                         "accepts_oracle": sum(t[4] for t in ro["trace"]),
                         "differing_decisions": diff, "differing_above_noise_floor": sig,
                         "rel_f": float(np.max(np.abs(rg.f - ro["f"])) / fs)}
        rows.append(row)
        print(json.dumps(row), flush=True)
    summ = {}
    for mode in ("literal", "stable"):
        att = sum(r[mode]["attempts"] for r in rows)
        dif = sum(len(r[mode]["differing_decisions"]) for r in rows)
        summ[mode] = {"seeds": S, "newton_attempts": att, "differing_decisions": dif,
                      "mismatch_rate": dif / max(att, 1),
                      "differing_above_noise_floor": sum(len(r[mode]["differing_above_noise_floor"]) for r in rows),
                      "seeds_with_equal_iteration_counts": sum(r[mode]["iterations_gpu"] == r[mode]["iterations_oracle"]
                                                               for r in rows),
                      "max_rel_f": max(r[mode]["rel_f"] for r in rows)}
    out = {"config": "C1 shape (n = m = 512, eps = 1e-2, ell = 10, tol 1e-9), seeds 1..%d; warm start and basis "
                     "from the oracle at eps' = 2e-2, shared" % S,
           "summary": summ, "seeds": rows}
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    json.dump(out, open(os.path.join(ROOT, "gpurun_out", "accept_modes_r02.json"), "w"), indent=1)
    print(json.dumps(summ, indent=1))


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 20)
