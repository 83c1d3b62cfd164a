"""Regenerate tests/golden/*.npz from the CPU oracle (oracle/sknr_oracle.cpp).

The reference cannot be built here (Eigen3 absent), so the golden vectors are
(1) the reference's own frozen known answers (test_core.cpp:31-46, :66-76,
support.hpp:87-101) and (2) oracle outputs on small seeded instances, pinned so
that a change in the oracle or in the GPU path is caught without rerunning the
oracle at test time. Run: python tests/golden/make_golden.py
"""
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))
import numpy as np

import oracle_ref as O
from paper_2506_14780_b200 import generators as G
from support import random_problem_data, random_vector


def main():
    out = {}
    # reference KATs (frozen 40-digit values from the reference's tests)
    out["kat_lse_values"] = np.array([0.3, -0.7, 1.1])
    out["kat_lse_expected"] = np.array([0.4804922094646261770])
    out["kat_2x2_g"] = np.array([0.3798854930417224754, 0.3798854930417224754])
    # C1 at n = m = 128: SK trajectory (40 iterations) and full solve
    inst = G.config("C1", n=128, m=128)
    P = O.Instance(inst.alpha, inst.beta, inst.epsilon, x=inst.x, y=inst.y)
    out["c1_x"], out["c1_y"] = inst.x, inst.y
    out["c1_alpha"], out["c1_beta"] = inst.alpha, inst.beta
    out["c1_eps"] = np.array([inst.epsilon])
    r = O.solve(P, tol=1e-30, max_iter=40)
    out["c1_sk40_f"], out["c1_sk40_g"] = r["f"], r["g"]
    out["c1_sk40_err"] = np.array([t[0] for t in r["trace"]])
    r = O.solve(P, tol=1e-9)
    out["c1_solve_f"], out["c1_solve_g"] = r["f"], r["g"]
    out["c1_solve_iters"] = np.array([r["iterations"]])
    f = np.linspace(-0.02, 0.02, 128)
    out["c1_f_probe"] = f
    out["c1_g_of_f"] = O.ctransform_of_f(P, f)
    # dense 7 x 9 random problem of test_solver.cpp:187-202 (seed 65, eps 0.5)
    rng = G.SplitMix64(65)
    cost, a, b = random_problem_data(rng, 7, 9)
    Pd = O.Instance(a, b, 0.5, cost=cost)
    r = O.solve(Pd, tol=1e-30, max_iter=40)
    out["d79_cost"], out["d79_alpha"], out["d79_beta"] = cost, a, b
    out["d79_f"], out["d79_g"] = r["f"], r["g"]
    out["d79_err"] = np.array([t[0] for t in r["trace"]])
    np.savez_compressed(os.path.join(HERE, "sknr_golden_v1.npz"), **out)
    print("wrote", os.path.join(HERE, "sknr_golden_v1.npz"), sorted(out))


if __name__ == "__main__":
    main()
