"""Opt-in fp32 variant (sknr_problem_set_precision(p, 32)): LSE sum passes with fp32
cell exponents and MUFU exp2 against the fp64 CPU oracle. North-star tolerance for an
fp32 variant: potentials and marginal error within 1e-5 relative; the solver's
stopping test still converges (the fp32 rounding is a fixed perturbation of the
kernel, see pts_f32_kernel), so iteration counts are compared too."""
import numpy as np
import pytest

import oracle_ref as O
import paper_2506_14780_b200 as sk
from paper_2506_14780_b200 import generators as G
from support import random_vector, rel_err

pytestmark = pytest.mark.gpu

TOL_F32 = 1e-5


def pair(inst, eps=None):
    eps = inst.epsilon if eps is None else eps
    gp = sk.PointProblem(inst.x, inst.y, inst.alpha, inst.beta, eps, inst.cost_scale)
    gp.set_precision(32)
    op = O.Instance(inst.alpha, inst.beta, eps, x=inst.x, y=inst.y, cost_div=1.0 / inst.cost_scale)
    return gp, op


@pytest.mark.parametrize("cfg,n,m,d", [("C1", 512, 512, 2), ("C2", 1500, 1300, 2), ("C3", 2000, 2013, 3),
                                       ("C4", 4096, 4096, 2)])
def test_fp32_transforms_match_oracle(cfg, n, m, d):
    inst = G.config(cfg, n=n, m=m)
    gp, op = pair(inst)
    f = random_vector(G.SplitMix64(7), n, 0.01)
    g_ref = O.ctransform_of_f(op, f)
    g32 = sk.ctransform_of_f(gp, f)
    assert rel_err(g32, g_ref) <= TOL_F32
    assert rel_err(sk.ctransform_of_g(gp, g_ref), O.ctransform_of_g(op, g_ref)) <= TOL_F32
    # and it really is another arithmetic than the fp64 path
    g64 = sk.ctransform_of_f(sk.PointProblem(inst.x, inst.y, inst.alpha, inst.beta, inst.epsilon,
                                             inst.cost_scale), f)
    assert not np.array_equal(g32, g64)


@pytest.mark.parametrize("d", [1, 4])
def test_fp32_other_dimensions(d):
    rng = np.random.default_rng(d)
    n, m = 700, 650
    x, y = rng.random((n, d)), rng.random((m, d))
    a, b = np.full(n, 1 / n), np.full(m, 1 / m)
    gp = sk.PointProblem(x, y, a, b, 2e-3)
    gp.set_precision(32)
    op = O.Instance(a, b, 2e-3, x=np.asfortranarray(x), y=np.asfortranarray(y))
    f = rng.standard_normal(n) * 1e-3
    assert rel_err(sk.ctransform_of_f(gp, f), O.ctransform_of_f(op, f)) <= TOL_F32


def test_fp32_sk_solve_matches_oracle():
    """C1 SK to 1e-9 (BASELINE configs[0]) and a C4-shaped 1024^2 problem at eps = 5e-4
    (the north-star eps, where the fp32 cell exponents are largest)."""
    for inst in (G.config("C1"), G.config("C4", n=1024, m=1024)):
        gp, op = pair(inst)
        r32 = sk.solve(gp, tol=1e-9)
        ro = O.solve(op, tol=1e-9, trace=False)
        assert r32.converged and ro["converged"]
        # the fp32 partial sums add potential-dependent rounding of ~1e-8 relative to
        # the column sums, i.e. ~1e-9 / sqrt(m / 512) to the marginal error: near
        # tol = 1e-9 the last few iterations can differ
        assert abs(r32.iterations - ro["iterations"]) <= 3 + ro["iterations"] // 100, (
            r32.iterations, ro["iterations"])
        assert rel_err(r32.f, ro["f"]) <= TOL_F32 and rel_err(r32.g, ro["g"]) <= TOL_F32
        # the fp64 marginal error of the fp32 potentials
        _, _, err, _ = O.plan_marginals(op, r32.f, r32.g)
        assert err <= 1e-5


def test_fp32_sknr_solve_matches_oracle():
    inst = G.config("C1")
    gp, op = pair(inst)
    warm = O.solve(op.with_epsilon(inst.basis_eps), tol=1e-9, trace=False)
    basis = O.top_modes(op.with_epsilon(inst.basis_eps), warm["f"], warm["g"], inst.ell)
    sb = sk.SpectralBasis(basis["vectors"], basis["vectors_sym"], basis["rhos"], inst.basis_eps)
    r32 = sk.solve(gp, tol=1e-9, ell=inst.ell, basis=sb, init=(warm["f"], warm["g"]))
    ro = O.solve(op, tol=1e-9, ell=inst.ell, V=basis["vectors"], init=(warm["f"], warm["g"]))
    assert r32.converged and ro["converged"]
    assert abs(r32.iterations - ro["iterations"]) <= 2
    assert rel_err(r32.f, ro["f"]) <= TOL_F32 and rel_err(r32.g, ro["g"]) <= TOL_F32


def test_fp32_is_deterministic_and_switchable():
    inst = G.config("C1")
    gp, _ = pair(inst)
    a, b = sk.solve(gp, tol=1e-9), sk.solve(gp, tol=1e-9)
    assert a.iterations == b.iterations and np.array_equal(a.f, b.f)
    gp.set_precision(64)
    ref = sk.solve(sk.PointProblem(inst.x, inst.y, inst.alpha, inst.beta, inst.epsilon), tol=1e-9)
    c = sk.solve(gp, tol=1e-9)
    assert c.iterations == ref.iterations and np.array_equal(c.f, ref.f)
    # with_epsilon keeps the precision
    q = gp.with_epsilon(0.02)
    assert getattr(q, "_precision", 64) == 64
    gp.set_precision(32)
    assert gp.with_epsilon(0.02)._precision == 32


def test_fp32_rejects_unsupported_problems():
    inst = G.config("C1", n=64, m=64)
    dense = sk.Problem(np.asfortranarray(np.abs(np.subtract.outer(inst.x[:, 0], inst.y[:, 0]))),
                       inst.alpha, inst.beta, 0.1)
    with pytest.raises(ValueError, match="set_precision"):
        sk._check(sk.lib().sknr_problem_set_precision(dense.handle, 32))
    gp, _ = pair(inst)
    with pytest.raises(ValueError, match="bits must be 32 or 64"):
        gp.set_precision(16)


def test_fp32_sharded_matches_unsharded():
    inst = G.config("C1", n=601, m=433)
    a, b = np.full(601, 1 / 601), np.full(433, 1 / 433)

    def mk():
        p = sk.PointProblem(inst.x, inst.y, a, b, inst.epsilon)
        p.set_precision(32)
        return p

    # the fp32 partial sums group the rows by shard, so (unlike fp64, 1e-12) the
    # sharded solve agrees with the unsharded one at the fp32 level
    ref = sk.solve(mk(), tol=1e-9)
    out = sk.run_emulated_shards(mk, 3, lambda p: sk.solve(p, tol=1e-9))
    for r in out:
        assert r.converged and abs(r.iterations - ref.iterations) <= 3 and rel_err(r.f, ref.f) <= TOL_F32
        assert np.array_equal(r.f, out[0].f)


def test_mufu_peak_is_measured():
    gex2, ms = sk.bench_mufu_peak()
    assert 1000.0 < gex2 < 20000.0 and ms > 0


def test_fp32_culled_matches_fp32_dense():
    """Both opt-ins together: culling (terms below e^-60 skipped) with the fp32 arithmetic
    on the kept groups; a 4096^2 C4-shaped problem at eps = 2e-3."""
    inst = G.config("C4", n=4096, m=4096)

    def mk(cull):
        p = sk.PointProblem(inst.x, inst.y, inst.alpha, inst.beta, 2e-3)
        p.set_precision(32)
        if cull:
            p.set_culling(60.0)
        return p

    ref = sk.solve(mk(False), tol=1e-9)
    pc = mk(True)
    r = sk.solve(pc, tol=1e-9)
    assert sk.debug_counters(pc)["cull_kept"] < sk.debug_counters(pc)["cull_tested"]
    assert r.converged, (r.iterations, ref.iterations)
    # fp32 group sums round differently from the dense kernel's: near tol the
    # stopping iteration can move by a few (as against the oracle, test above)
    assert abs(r.iterations - ref.iterations) <= 3 + ref.iterations // 100, (r.iterations, ref.iterations)
    assert rel_err(r.f, ref.f) <= 1e-6 and rel_err(r.g, ref.g) <= 1e-6
    op = O.Instance(inst.alpha, inst.beta, 2e-3, x=inst.x, y=inst.y)
    f = random_vector(G.SplitMix64(3), inst.n, 0.01)
    assert rel_err(sk.ctransform_of_f(pc, f), O.ctransform_of_f(op, f)) <= TOL_F32
