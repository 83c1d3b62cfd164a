"""Pins the CPU oracle (oracle/sknr_oracle.cpp) to the reference's own
known-answer tests for this path (proj/tests/test_core.cpp, test_solver.cpp,
test_spectral.cpp, support.hpp). CPU only."""
import math

import numpy as np
import pytest

import oracle_ref as O
from support import (gauge_normalized, projector_distance, random_measure, random_problem_data,
                     random_vector, symmetric_2x2, symmetric_2x2_optimum)
from paper_2506_14780_b200.generators import SplitMix64


def test_log_sum_exp_basics():  # test_core.cpp:13-29
    assert abs(O.log_sum_exp([0.0, 0.0], [math.log(0.5)] * 2)) <= 1e-15
    assert O.log_sum_exp([1000.0, 1000.0], [0.0, 0.0]) == pytest.approx(1000.0 + math.log(2.0),
                                                                        rel=1e-15)
    assert math.isfinite(O.log_sum_exp([1e300, 1e300], [0.0, 0.0]))
    with pytest.raises(ValueError, match="empty reduction"):
        O.log_sum_exp([], [])


def test_log_sum_exp_frozen_value():  # test_core.cpp:31-46
    lw = math.log(1.0 / 3.0)
    got = O.log_sum_exp([0.3, -0.7, 1.1], [lw] * 3)
    assert got == pytest.approx(0.4804922094646261770, rel=1e-15)


def test_ctransform_2x2_frozen():  # test_core.cpp:66-76
    cost, a, b = symmetric_2x2()
    P = O.Instance(a, b, 1.0, cost=cost)
    g = O.ctransform_of_f(P, np.zeros(2))
    assert g == pytest.approx([0.3798854930417224754] * 2, rel=1e-15)
    f = O.ctransform_of_g(P, g)
    assert np.max(np.abs(f)) <= 1e-15


def test_zero_cost_plan_is_outer_product_exactly():  # test_core.cpp:101-113
    rng = SplitMix64(13)
    a = random_measure(rng, 3)
    b = random_measure(rng, 5)
    P = O.Instance(a, b, 0.9, cost=np.zeros((3, 5)))
    plan = O.coupling(P, np.zeros(3), np.zeros(5))
    assert np.max(np.abs(plan - np.outer(a, b))) == 0.0


def test_integer_gauge_shift_bitwise():  # test_core.cpp:115-122
    rng = SplitMix64(13)
    random_measure(rng, 3)
    random_measure(rng, 5)
    cost, a, b = random_problem_data(rng, 4, 4)
    P = O.Instance(a, b, 1.0, cost=cost)
    f = np.array([1.0, -2.0, 0.0, 3.0])
    g = np.array([2.0, 0.0, -1.0, 1.0])
    assert np.array_equal(O.coupling(P, f, g), O.coupling(P, f + 2.0, g - 2.0))


def test_column_exactness():  # test_core.cpp:174-184
    rng = SplitMix64(15)
    for _ in range(10):
        eps = 0.2 + rng.uniform01()
        cost, a, b = random_problem_data(rng, 6, 5)
        P = O.Instance(a, b, eps, cost=cost)
        f = random_vector(rng, 6, 2.0)
        g = O.ctransform_of_f(P, f)
        col = O.coupling(P, f, g).sum(axis=0)
        assert np.max(np.abs(col - b)) <= 1e-12


def test_overflow_safety():  # test_core.cpp:186-202
    rng = SplitMix64(16)
    cost = np.empty((6, 7), order="F")
    for j in range(7):
        for i in range(6):
            cost[i, j] = 1e4 * rng.uniform01()
    a = random_measure(rng, 6)
    b = random_measure(rng, 7)
    P = O.Instance(a, b, 1e-3, cost=cost)
    g = O.ctransform_of_f(P, np.zeros(6))
    f2 = O.ctransform_of_g(P, g)
    assert np.all(np.isfinite(g)) and np.all(np.isfinite(f2))


def test_sk_fixed_point_2x2():  # test_solver.cpp:91-96
    cost, a, b = symmetric_2x2()
    P = O.Instance(a, b, 1.0, cost=cost)
    f0, g0 = symmetric_2x2_optimum()
    r = O.solve(P, tol=1e-14, max_iter=3, init=(f0, g0))
    f, g = gauge_normalized(a, r["f"], r["g"])
    assert np.max(np.abs(f - f0)) <= 1e-12 and np.max(np.abs(g - g0)) <= 1e-12


def _reference_sk(cost, a, b, eps, iters):
    """Independent log-domain SK of test_solver.cpp:25-73 (numpy restatement)."""
    n, m = cost.shape
    f = np.zeros(n)
    g = np.zeros(m)
    errs = []
    for _ in range(iters):
        E = np.log(a)[:, None] + (f[:, None] - cost) / eps
        sh = E.max(axis=0)
        g = -eps * (sh + np.log(np.exp(E - sh).sum(axis=0)))
        E = np.log(b)[None, :] + (g[None, :] - cost) / eps
        sh = E.max(axis=1)
        f = -eps * (sh + np.log(np.exp(E - sh[:, None]).sum(axis=1)))
        c = a @ f
        f, g = f - c, g + c
        p = a[:, None] * b[None, :] * np.exp((f[:, None] + g[None, :] - cost) / eps)
        errs.append(np.linalg.norm(p.sum(1) - a) + np.linalg.norm(p.sum(0) - b))
    return f, g, errs


def test_solve_reproduces_reference_sk_trajectory():  # test_solver.cpp:187-202
    rng = SplitMix64(65)
    cost, a, b = random_problem_data(rng, 7, 9)
    P = O.Instance(a, b, 0.5, cost=cost)
    r = O.solve(P, tol=1e-30, max_iter=40)
    f, g, errs = _reference_sk(cost, a, b, 0.5, 40)
    assert np.max(np.abs(r["f"] - f)) <= 1e-14
    assert np.max(np.abs(r["g"] - g)) <= 1e-14
    assert len(r["trace"]) == 40
    for k in range(40):
        assert abs(r["trace"][k][0] - errs[k]) <= 1e-12


def test_solve_converges_and_max_iter_not_error():  # test_solver.cpp:204-219
    rng = SplitMix64(66)
    cost, a, b = random_problem_data(rng, 6, 8)
    P = O.Instance(a, b, 1.0, cost=cost)
    r = O.solve(P, tol=1e-10)
    assert r["converged"]
    plan = O.coupling(P, r["f"], r["g"])
    err = np.linalg.norm(plan.sum(1) - a) + np.linalg.norm(plan.sum(0) - b)
    assert err <= 1e-10
    r2 = O.solve(P, tol=1e-14, max_iter=2)
    assert not r2["converged"] and r2["iterations"] == 2


def _dense_svd_basis(cost, a, b, eps, f, g, ell):  # support.hpp:61-76 with numpy SVD
    blk = np.sqrt(a)[:, None] * np.exp((f[:, None] + g[None, :] - cost) / eps) * np.sqrt(b)[None, :]
    U, s, _ = np.linalg.svd(blk)
    vs = U[:, 1:1 + ell]
    return vs / np.sqrt(a)[:, None], vs, s[1:1 + ell]


def test_top_modes_matches_dense_svd():  # test_spectral.cpp (top_modes vs dense SVD, 1e-8)
    rng = SplitMix64(44)
    cost, a, b = random_problem_data(rng, 12, 10)
    P = O.Instance(a, b, 0.4, cost=cost)
    r = O.solve(P, tol=1e-13)
    ell = 3
    tm = O.top_modes(P, r["f"], r["g"], ell)
    _, vs, rho = _dense_svd_basis(cost, a, b, 0.4, r["f"], r["g"], ell)
    assert np.max(np.abs(tm["rhos"] - rho)) <= 1e-8
    assert np.max(np.abs(tm["vectors_sym"].T @ tm["vectors_sym"] - np.eye(ell))) <= 1e-10
    assert np.max(np.abs(np.sqrt(a) @ tm["vectors_sym"])) <= 1e-9
    assert projector_distance(vs, tm["vectors_sym"]) <= 1e-6


def test_newton_reduces_iterations_and_monotone_values():  # test_solver.cpp:221-259
    rng = SplitMix64(67)
    cost, a, b = random_problem_data(rng, 10, 8)
    eps = 0.15
    P = O.Instance(a, b, eps, cost=cost)
    ref = O.solve(P, tol=1e-13)
    V, _, _ = _dense_svd_basis(cost, a, b, eps, ref["f"], ref["g"], 3)
    plain = O.solve(P, tol=1e-11)
    fast = O.solve(P, tol=1e-11, ell=3, V=V)
    assert fast["converged"] and plain["converged"]
    assert fast["iterations"] <= plain["iterations"]
    vals = [t[2] for t in fast["trace"]]
    assert all(vals[k] >= vals[k - 1] - 1e-12 for k in range(1, len(vals)))


def test_restricted_derivatives_match_finite_differences():  # test_objective.cpp:142-179
    rng = SplitMix64(71)
    cost, a, b = random_problem_data(rng, 9, 7)
    P = O.Instance(a, b, 0.6, cost=cost)
    f = random_vector(rng, 9, 0.5)
    V = np.asfortranarray(np.array([random_vector(rng, 9) for _ in range(3)]).T)
    g = O.ctransform_of_f(P, f)
    grad, hess = O.restricted_derivatives(P, f, g, V)
    h = 1e-5
    for c in range(3):
        up = O.semi_dual_value(P, f + h * V[:, c])
        dn = O.semi_dual_value(P, f - h * V[:, c])
        assert abs((up - dn) / (2 * h) - grad[c]) <= 1e-7
    assert np.max(np.abs(hess - hess.T)) == 0.0
    assert np.all(np.linalg.eigvalsh(hess) <= 1e-12)


def test_output_parallel_is_bitwise_identical():
    rng = SplitMix64(5)
    cost, a, b = random_problem_data(rng, 37, 29)
    P = O.Instance(a, b, 0.05, cost=cost)
    f = random_vector(rng, 37, 0.3)
    O.set_threads(1)
    g1 = O.ctransform_of_f(P, f)
    f1 = O.ctransform_of_g(P, g1)
    O.set_threads(4)
    g4 = O.ctransform_of_f(P, f)
    f4 = O.ctransform_of_g(P, g4)
    O.set_threads(1)
    assert np.array_equal(g1, g4) and np.array_equal(f1, f4)


def test_points_kind_matches_dense_cost():
    rng = SplitMix64(9)
    x = np.asfortranarray(np.array([[rng.uniform01() for _ in range(3)] for _ in range(11)]))
    y = np.asfortranarray(np.array([[rng.uniform01() for _ in range(3)] for _ in range(13)]))
    a = random_measure(rng, 11)
    b = random_measure(rng, 13)
    cost = np.asfortranarray(((x[:, None, :] - y[None, :, :]) ** 2).sum(-1))
    Pd = O.Instance(a, b, 0.05, cost=cost)
    Pp = O.Instance(a, b, 0.05, x=x, y=y)
    f = random_vector(rng, 11, 0.1)
    assert np.max(np.abs(O.ctransform_of_f(Pd, f) - O.ctransform_of_f(Pp, f))) <= 1e-14


@pytest.mark.parametrize("k_sk", [1, 2, 3, 4, 6])
def test_stable_delta_q_matches_literal_gain(k_sk):
    """The stable accept test evaluates Q(f') - Q(f) directly (sknr_oracle.cpp
    stable_delta_q); wherever the literal difference is well above Q's rounding the two
    must agree -- including large steps (|d|/eps up to the 600 literal-fallback span) that
    move a column's mass away, where log1p(t/s) would cancel to -inf (t/s -> -1) and the
    log(u/s) form takes over. BASELINE C3 shape (d = 3, Dirichlet weights, eps = 1e-3)."""
    from paper_2506_14780_b200 import generators as G
    from support import smooth_basis

    c = G.config("C3", n=500, m=450)
    P = O.Instance(c.alpha, c.beta, c.epsilon, x=c.x, y=c.y, cost_div=1.0 / c.cost_scale)
    r0 = O.solve(P, tol=1e-300, max_iter=k_sk)
    V = smooth_basis(c.x, c.alpha, c.ell)
    gains = {}
    for mode in ("literal", "stable"):
        with O.accept_mode(mode):
            r = O.solve(P, tol=1e-300, max_iter=1, ell=c.ell, V=V, init=(r0["f"], r0["g"]))
        gains[mode] = r["trace"][0]
    lit, st = gains["literal"], gains["stable"]
    step_over_eps = lit[6] / c.epsilon
    assert math.isfinite(st[5]) and math.isfinite(st[2])
    q_ulp = 4 * np.spacing(abs(lit[2]))
    assert abs(st[5] - lit[5]) <= 1e-9 * abs(lit[5]) + q_ulp, (step_over_eps, st[5], lit[5])
    assert st[4] == lit[4]
