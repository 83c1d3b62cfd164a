"""Golden fixtures (tests/golden/sknr_golden_v1.npz, made by
tests/golden/make_golden.py from the reference KATs and the CPU oracle).
CPU tests pin the oracle to them; GPU tests compare the B200 path to them
without running the oracle."""
import os

import numpy as np
import pytest

import oracle_ref as O

GOLD = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "sknr_golden_v1.npz"))


def test_oracle_reproduces_golden_kats():
    lw = np.log(np.full(3, 1.0 / 3.0))
    assert O.log_sum_exp(GOLD["kat_lse_values"], lw) == pytest.approx(GOLD["kat_lse_expected"][0], rel=1e-15)
    cost = np.array([[0.0, 1.0], [1.0, 0.0]])
    P = O.Instance([0.5, 0.5], [0.5, 0.5], 1.0, cost=cost)
    assert np.allclose(O.ctransform_of_f(P, np.zeros(2)), GOLD["kat_2x2_g"], rtol=1e-15, atol=0)


def test_oracle_reproduces_golden_trajectories():
    P = O.Instance(GOLD["c1_alpha"], GOLD["c1_beta"], GOLD["c1_eps"][0], x=GOLD["c1_x"], y=GOLD["c1_y"])
    r = O.solve(P, tol=1e-30, max_iter=40)
    assert np.array_equal(r["f"], GOLD["c1_sk40_f"])  # the oracle is deterministic bitwise
    Pd = O.Instance(GOLD["d79_alpha"], GOLD["d79_beta"], 0.5, cost=GOLD["d79_cost"])
    r = O.solve(Pd, tol=1e-30, max_iter=40)
    assert np.array_equal(r["f"], GOLD["d79_f"])


@pytest.mark.gpu
def test_gpu_matches_golden():
    import paper_2506_14780_b200 as sk

    rel = lambda a, b: float(np.max(np.abs(a - b)) / np.max(np.abs(b)))
    p = sk.PointProblem(GOLD["c1_x"], GOLD["c1_y"], GOLD["c1_alpha"], GOLD["c1_beta"], GOLD["c1_eps"][0])
    assert rel(sk.ctransform_of_f(p, GOLD["c1_f_probe"]), GOLD["c1_g_of_f"]) <= 1e-12
    r = sk.solve(p, tol=1e-30, max_iter=40)
    assert rel(r.f, GOLD["c1_sk40_f"]) <= 1e-12 and rel(r.g, GOLD["c1_sk40_g"]) <= 1e-12
    errs = np.array([t.marginal_error for t in r.trace])
    assert np.max(np.abs(errs - GOLD["c1_sk40_err"]) / GOLD["c1_sk40_err"]) <= 1e-9
    r = sk.solve(p, tol=1e-9)
    assert r.iterations == int(GOLD["c1_solve_iters"][0])
    assert rel(r.f, GOLD["c1_solve_f"]) <= 1e-9
    d = sk.Problem(GOLD["d79_cost"], GOLD["d79_alpha"], GOLD["d79_beta"], 0.5)
    r = sk.solve(d, tol=1e-30, max_iter=40)
    assert np.max(np.abs(r.f - GOLD["d79_f"])) <= 1e-14
    assert np.max(np.abs(np.array([t.marginal_error for t in r.trace]) - GOLD["d79_err"])) <= 1e-12
