"""GPU checks of the rest of the reference API surface (SinkhornOperator apply_R /
apply_Rt, dual_value, semi_dual_hessian_quadform, newton_step, sk_sweep,
spectrum_report, projector_distance, streamed coupling, harness oracle_solve /
full_semi_dual_hessian, and the CLI) against the CPU oracle and the reference's
own closed-form tests."""
import os

import numpy as np
import pytest

import oracle_ref as O
import paper_2506_14780_b200 as sk
from paper_2506_14780_b200 import cli
from paper_2506_14780_b200 import generators as G
from paper_2506_14780_b200 import harness as H
from paper_2506_14780_b200 import io as sio
from support import (projector_distance, random_problem_data, random_vector, rel_err, symmetric_2x2,
                     symmetric_2x2_optimum)

pytestmark = pytest.mark.gpu


def dense_pair(seed, n, m, eps):
    rng = G.SplitMix64(seed)
    cost, a, b = random_problem_data(rng, n, m)
    return sk.Problem(cost, a, b, eps), O.Instance(a, b, eps, cost=cost), rng


def points_pair(seed, n, m, d, eps):
    r = np.random.default_rng(seed)
    x = np.asfortranarray(r.uniform(0, 1, (n, d)))
    y = np.asfortranarray(r.uniform(0, 1, (m, d)))
    a = r.uniform(0.5, 1.5, n)
    a /= a.sum()
    b = r.uniform(0.5, 1.5, m)
    b /= b.sum()
    return sk.PointProblem(x, y, a, b, eps), O.Instance(a, b, eps, x=x, y=y), r


@pytest.mark.parametrize("kind", ["dense", "points"])
def test_apply_R_and_Rt_match_oracle(kind):  # spectral.cpp:29-66
    if kind == "dense":
        gp, op, rng = dense_pair(11, 150, 97, 0.1)
        f = random_vector(rng, 150, 0.1)
        g1 = random_vector(rng, 97)
        f1 = random_vector(rng, 150)
    else:
        gp, op, r = points_pair(12, 300, 211, 3, 0.02)
        f = r.uniform(-0.05, 0.05, 300)
        g1 = r.standard_normal(211)
        f1 = r.standard_normal(300)
    g = O.ctransform_of_f(op, f)
    assert rel_err(sk.apply_R(gp, f, g, g1), O.apply_R(op, f, g, g1)) <= 1e-12
    assert rel_err(sk.apply_Rt(gp, f, g, f1), O.apply_Rt(op, f, g, f1)) <= 1e-12
    rk, rtk = sk.apply_K(gp, f, g, f1, g1)
    assert rel_err(rk, O.apply_R(op, f, g, g1)) <= 1e-12 and rel_err(rtk, O.apply_Rt(op, f, g, f1)) <= 1e-12
    with pytest.raises(ValueError, match="length mismatch"):
        sk.apply_R(gp, f, g, f1)


@pytest.mark.parametrize("kind", ["dense", "points"])
def test_dual_value_matches_oracle(kind):  # objective.cpp:10-40
    gp, op, _ = dense_pair(21, 64, 80, 0.2) if kind == "dense" else points_pair(22, 200, 150, 2, 0.05)
    r = sk.solve(gp, tol=1e-12)
    for f, g in [(r.f, r.g), (r.f + 0.01, r.g - 0.02)]:
        v_gpu = sk.dual_value(gp, f, g)
        v_ref = O.dual_value(op, f, g)
        assert abs(v_gpu - v_ref) <= 1e-12 * max(1.0, abs(v_ref))
    # at the optimum the dual equals the semi-dual (total mass 1)
    assert abs(sk.dual_value(gp, r.f, r.g) - sk.semi_dual_value(gp, r.f)) <= 1e-9
    with pytest.raises(ValueError, match="finite"):
        sk.dual_value(gp, np.full(gp.n, np.nan), r.g)


def test_hessian_quadform_matches_oracle_and_dense_hessian():  # test_objective.cpp:190-205
    rng = G.SplitMix64(29)
    cost, a, b = random_problem_data(rng, 7, 9, 1.0)
    gp = sk.Problem(cost, a, b, 0.6)
    op = O.Instance(a, b, 0.6, cost=cost)
    f = random_vector(rng, 7, 0.5)
    hess = H.full_semi_dual_hessian(gp, f)
    assert np.max(np.abs(hess @ np.ones(7))) <= 1e-12
    for _ in range(20):
        u = random_vector(rng, 7)
        direct = sk.semi_dual_hessian_quadform(gp, f, u)
        assert abs(direct - O.semi_dual_hessian_quadform(op, f, u)) <= 1e-12 * abs(direct)
        assert abs(u @ hess @ u - direct) <= 1e-12 * abs(direct)
    with pytest.raises(ValueError, match="dense Hessian too large"):
        H.full_semi_dual_hessian(gp, f, 5)


def test_2x2_hessian_spectrum_closed_form():  # test_objective.cpp:207-223, support.hpp:87-101
    eps = 0.7
    cost, a, b = symmetric_2x2()
    gp = sk.Problem(cost, a, b, eps)
    f, g = symmetric_2x2_optimum(eps)
    hess = H.full_semi_dual_hessian(gp, f)
    hs = np.diag(1 / np.sqrt(a)) @ hess @ np.diag(1 / np.sqrt(a))
    ev = np.linalg.eigvalsh(hs)
    rho = np.tanh(1.0 / (2 * eps))
    assert abs(ev[0] - (-(1 - rho ** 2) / eps)) <= 1e-9 * abs(ev[0])
    assert abs(ev[1]) <= 1e-9
    rep = sk.spectrum(gp, f, g, 1, vectors=True)
    assert abs(rep["rho"][0] - rho) <= 1e-10
    assert abs(rep["hessian_eigs_low"][0] - (1 - rho) / eps) <= 1e-9
    assert abs(rep["hessian_eigs_high"][0] - (1 + rho) / eps) <= 1e-9
    assert rep["eigenvalues_of_K"][0] == (rep["rho"][0], -rep["rho"][0])
    # restricted Hessian in the exact eigenbasis (test_objective.cpp:181-188)
    basis = sk.top_modes(gp, f, g, 1)
    _, hr = sk.restricted_derivatives(gp, f, basis, g)
    assert abs(hr[0, 0] - (-(1 - basis.rhos[0] ** 2) / eps)) <= 1e-8 * abs(hr[0, 0])
    with pytest.raises(ValueError, match="need 1 <= k"):
        sk.spectrum(gp, f, g, 2)


def test_spectrum_vectors_match_oracle():  # spectral.cpp:195-228
    gp, op, _ = dense_pair(41, 120, 90, 0.2)
    r = O.solve(op, tol=1e-12)
    k = 5
    rep = sk.spectrum(gp, r["f"], r["g"], k, vectors=True)
    ob = O.top_modes(op, r["f"], r["g"], k)
    assert rel_err(rep["rho"], ob["rhos"]) <= 1e-8
    assert projector_distance(np.sqrt(op.alpha)[:, None] * rep["vectors_f"], ob["vectors_sym"]) <= 1e-6
    vs = O.apply_sym_t_block(op, r["f"], r["g"], ob["vectors_sym"])
    vg_ref = vs / ob["rhos"][None, :] / np.sqrt(op.beta)[:, None]
    for c in range(k):  # eigenvector signs are arbitrary
        s = np.sign(rep["vectors_g"][:, c] @ vg_ref[:, c])
        assert rel_err(s * rep["vectors_g"][:, c], vg_ref[:, c]) <= 1e-6


def test_projector_distance():  # spectral.cpp:230-242
    r = np.random.default_rng(5)
    A = np.linalg.qr(r.standard_normal((200, 6)))[0]
    B = np.linalg.qr(A + 1e-3 * r.standard_normal((200, 6)))[0]
    ba = sk.SpectralBasis(A, A, np.zeros(6), 0.1)
    bb = sk.SpectralBasis(B, B, np.zeros(6), 0.1)
    assert abs(sk.projector_distance(ba, bb) - projector_distance(A, B)) <= 1e-12
    assert sk.projector_distance(ba, ba) <= 1e-7
    C = np.linalg.qr(r.standard_normal((200, 5)))[0]
    with pytest.raises(ValueError, match="dimension mismatch"):
        sk.projector_distance(ba, sk.SpectralBasis(C, C, np.zeros(5), 0.1))


def test_newton_step_and_sk_sweep_match_oracle():  # solver.cpp:12-17, :59-69
    gp, op, r = points_pair(51, 400, 300, 2, 0.01)
    f0 = O.solve(op, tol=1e-4)["f"]
    V = np.asfortranarray(np.linalg.qr(r.standard_normal((400, 6)))[0])
    out = sk.newton_step(gp, f0, sk.SpectralBasis(V, V, np.zeros(6), 0.01))
    fo, acc, fail = O.newton_step(op, f0, V)
    assert out.accepted == acc and out.factorization_failed == fail
    assert rel_err(out.f, fo) <= 1e-9
    f1, g1 = sk.sk_sweep(gp, f0)
    g_ref = O.ctransform_of_f(op, f0)
    assert rel_err(g1, g_ref) <= 1e-12 and rel_err(f1, O.ctransform_of_g(op, g_ref)) <= 1e-12
    with pytest.raises(ValueError, match="empty basis"):
        sk.newton_step(gp, f0, sk.SpectralBasis(np.zeros((400, 0)), np.zeros((400, 0)), np.zeros(0), 0.01))


def test_coupling_rows_and_streamed_csv(tmp_path):  # core.cpp:84-112, main.cpp:149-154
    gp, op, rng = dense_pair(61, 37, 23, 0.3)
    r = sk.solve(gp, tol=1e-11)
    plan = sk.coupling(gp, r.f, r.g)
    assert rel_err(plan, O.coupling(op, r.f, r.g)) <= 1e-13
    assert np.array_equal(sk.coupling_rows(gp, r.f, r.g, 5, 19), plan[5:19])
    path = str(tmp_path / "coupling.csv")
    err = sio.write_coupling_csv(path, gp, r.f, r.g, block_bytes=8 * 23 * 4)
    back = sio.read_csv_matrix(path)
    assert np.array_equal(back, plan)  # %.17g round-trips bitwise
    assert abs(err - sk.marginal_error(gp, plan)) <= 1e-15
    with pytest.raises(ValueError, match="row range"):
        sk.coupling_rows(gp, r.f, r.g, 10, 40)


def test_oracle_solve_ground_truth():  # oracle.cpp:21-90
    gp, op, _ = dense_pair(71, 40, 50, 0.05)
    sol = H.oracle_solve(gp, 1e-12)
    assert sol.residual <= 1e-11 and sol["residual"] == sol.residual
    ref = O.solve(op, tol=1e-13)
    c = float(op.alpha @ ref["f"])
    assert rel_err(sol.f, ref["f"] - c) <= 1e-9
    assert abs(float(op.alpha @ sol.f)) <= 1e-15


def test_cli_solve_spectrum_anneal(tmp_path, capsys):  # main.cpp:120-218
    r = np.random.default_rng(3)
    src = tmp_path / "src.csv"
    tgt = tmp_path / "tgt.csv"
    xs = r.uniform(0, 1, (60, 2))
    yt = r.uniform(0, 1, (70, 2))
    w = r.uniform(0.5, 1.5, 70)
    np.savetxt(src, xs, delimiter=",", fmt="%.17g")
    with open(tgt, "w") as fh:
        fh.write("x,y,weight\n")
        for p, wi in zip(yt, w):
            fh.write(f"{float(p[0])!r},{float(p[1])!r},{float(wi)!r}\n")
    out = tmp_path / "solve"
    rc = cli.main(["solve", "--points", str(src), str(tgt), "--epsilon", "0.05", "--ell", "4",
                   "--basis-from", "0.1", "--out", str(out)])
    text = capsys.readouterr()
    assert rc == 0, text
    assert "weights renormalized" in text.err
    assert text.out.startswith("converged=true iters=")
    for name in ("potentials.csv", "coupling.csv", "trace.csv"):
        assert os.path.exists(out / name)
    pots = open(out / "potentials.csv").read().splitlines()
    assert pots[0] == "which,index,value" and len(pots) == 1 + 60 + 70
    # same result through the library
    gp = sk.PointProblem(xs, yt, np.full(60, 1 / 60), w / w.sum(), 0.05)
    f_cli = np.array([float(line.split(",")[2]) for line in pots[1:61]])
    warm = sk.solve(gp.with_epsilon(0.1))
    basis = sk.top_modes(gp.with_epsilon(0.1), warm.f, warm.g, 4)
    res = sk.solve(gp, ell=4, basis=basis, init=(warm.f, warm.g))
    assert np.array_equal(f_cli, res.f)
    rc = cli.main(["spectrum", "--synthetic", "gauss2d", "--n", "30", "--m", "40", "--epsilons", "0.5,0.25",
                   "--k", "3", "--vectors", "--out", str(tmp_path / "spec")])
    assert rc == 0
    assert os.path.exists(tmp_path / "spec" / "spectrum_001.json")
    rc = cli.main(["anneal", "--synthetic", "two_moons", "--n", "40", "--m", "40", "--schedule", "0.2,0.1,0.05",
                   "--warm", "spectral", "--ell", "3", "--out", str(tmp_path / "ann")])
    assert rc == 0
    assert open(tmp_path / "ann" / "anneal_trace.csv").readline().startswith("stage,epsilon,iter,")
    rc = cli.main(["solve", "--synthetic", "gauss2d", "--epsilon", "0.01", "--max-iter", "3",
                   "--out", str(tmp_path / "capped")])
    assert rc == 2


def test_cli_opt_in_flags(tmp_path, capsys):
    """--cull / --warm-fp32 / --basis-method (additions beyond the reference CLI) give the
    reference pipeline's potentials to the solve tolerance's resolution."""
    base = ["solve", "--synthetic", "gauss2d", "--n", "300", "--m", "280", "--epsilon", "0.01", "--ell", "6",
            "--basis-from", "0.02", "--no-trace"]
    assert cli.main(base + ["--out", str(tmp_path / "ref")]) == 0
    assert cli.main(base + ["--cull", "60", "--warm-fp32", "--basis-method", "lanczos",
                            "--out", str(tmp_path / "opt")]) == 0
    out = capsys.readouterr().out.splitlines()
    assert all(line.startswith("converged=true") for line in out[-2:])
    read = lambda d: np.array([float(l.split(",")[2]) for l in open(tmp_path / d / "potentials.csv").read()
                               .splitlines()[1:]])
    assert rel_err(read("opt"), read("ref")) <= 1e-7
    np.savetxt(tmp_path / "c.csv", np.ones((3, 3)), delimiter=",")
    rc = cli.main(["solve", "--cost", str(tmp_path / "c.csv"), "--epsilon", "0.5", "--cull", "60", "--out",
                   str(tmp_path / "x")])
    assert rc == 1 and "point-cloud" in capsys.readouterr().err


def test_cli_zero_cost_exact_outer_product(tmp_path):  # test_cli.cpp:74-90
    (tmp_path / "zero3x3.csv").write_text("0,0,0\n0,0,0\n0,0,0\n")
    rc = cli.main(["solve", "--cost", str(tmp_path / "zero3x3.csv"), "--epsilon", "0.5", "--out",
                   str(tmp_path / "out")])
    assert rc == 0
    plan = sio.read_csv_matrix(str(tmp_path / "out" / "coupling.csv"))
    w = 1.0 / 3.0
    assert np.all(plan == w * w)


def test_cli_spectrum_round_trip_and_single_stage_anneal(tmp_path, capsys):  # test_cli.cpp:159-203
    import json
    rc = cli.main(["spectrum", "--synthetic", "gauss2d", "--n", "30", "--m", "40", "--epsilons", "0.5",
                   "--k", "4", "--out", str(tmp_path / "s")])
    assert rc == 0
    line = capsys.readouterr().out.strip()
    rep = json.load(open(tmp_path / "s" / "spectrum_000.json"))
    assert len(rep["rho"]) == 4 and rep["k"] == 4
    assert line.endswith("file=spectrum_000.json")
    assert float(line.split("rho_1=")[1].split()[0]) == rep["rho"][0]  # bitwise through %.17g
    rc = cli.main(["anneal", "--synthetic", "gauss2d", "--n", "30", "--m", "40", "--schedule", "0.2",
                   "--out", str(tmp_path / "a")])
    assert rc == 0
    x, a, y, b = G.make_instance("gauss2d", 30, 40)
    ref = sk.solve(sk.PointProblem(x, y, a, b, 0.2))
    rows = open(tmp_path / "a" / "stage_00_potentials.csv").read().splitlines()[1:31]
    assert np.array_equal([float(r.split(",")[2]) for r in rows], ref.f)


def test_solve_batch_is_bitwise_identical_to_single_solves():
    probs, bases, inits = [], [], []
    for s in range(6):
        if s % 3 == 2:
            gp, _, _ = dense_pair(100 + s, 90 + 7 * s, 70 + 5 * s, 0.05)
        else:
            gp, _, _ = points_pair(100 + s, 200 + 31 * s, 150 + 17 * s, 1 + s % 4, 0.02)
        probs.append(gp)
        warm = sk.solve(gp.with_epsilon(0.04))
        bases.append(sk.top_modes(gp.with_epsilon(0.04), warm.f, warm.g, 5))
        inits.append((warm.f, warm.g))
    for ell in (0, 5):
        kw = dict(tol=1e-10, ell=ell, bases=bases if ell else None, inits=inits)
        res = sk.solve_batch(probs, **kw)
        for p, r, b, i in zip(probs, res, bases, inits):
            one = sk.solve(p, tol=1e-10, ell=ell, basis=b if ell else None, init=i)
            assert r.converged and r.iterations == one.iterations
            assert np.array_equal(r.f, one.f) and np.array_equal(r.g, one.g)
    with pytest.raises(ValueError, match="duplicate problem handle"):
        sk.solve_batch([probs[0], probs[0]])
    with pytest.raises(ValueError, match="requires a basis"):
        sk.solve_batch(probs, ell=5)


@pytest.mark.parametrize("d,n,m", [(1, 5000, 9000), (2, 9000, 5000), (3, 4100, 6000), (4, 2100, 4500)])
def test_culled_transforms_match_oracle(d, n, m):
    """Opt-in culling (sknr_problem_set_culling): Morton-ordered group bounds skip terms
    below e^-60 of each output's total; ragged sizes exercise partial groups."""
    r = np.random.default_rng(d * 31 + n)
    x = np.asfortranarray(r.uniform(0, 1, (n, d)))
    y = np.asfortranarray(r.uniform(0, 1, (m, d)))
    a = np.full(n, 1.0 / n)
    b = np.full(m, 1.0 / m)
    eps = 2e-3
    gp = sk.PointProblem(x, y, a, b, eps)
    gp.set_culling(60.0)
    op = O.Instance(a, b, eps, x=x, y=y)
    f = 0.01 * r.standard_normal(n)
    g_ref = O.ctransform_of_f(op, f)
    assert rel_err(sk.ctransform_of_f(gp, f), g_ref) <= 1e-12
    assert rel_err(sk.ctransform_of_g(gp, g_ref), O.ctransform_of_g(op, g_ref)) <= 1e-12
    # solver path (bound shift + culling) against the dense path
    gd = sk.PointProblem(x, y, a, b, eps)
    rc = sk.solve(gp, tol=1e-9, max_iter=400, trace=False)
    rd = sk.solve(gd, tol=1e-9, max_iter=400, trace=False)
    assert rc.iterations == rd.iterations and rc.converged == rd.converged
    assert rel_err(rc.f, rd.f) <= 1e-12 and rel_err(rc.g, rd.g) <= 1e-12


def test_culling_errors_and_off_switch():
    gp, _, _ = dense_pair(5, 40, 30, 0.1)
    with pytest.raises(ValueError, match="point-cloud problem"):
        lib_set = sk.lib().sknr_problem_set_culling
        sk._check(lib_set(gp.handle, 60.0))
    pp, _, _ = points_pair(6, 3000, 2500, 2, 0.01)
    with pytest.raises(ValueError, match="threshold below 40"):
        pp.set_culling(10.0)
    f = np.zeros(3000)
    g0 = sk.ctransform_of_f(pp, f)
    pp.set_culling(60.0)
    g1 = sk.ctransform_of_f(pp, f)
    pp.set_culling(0.0)
    assert np.array_equal(sk.ctransform_of_f(pp, f), g0)
    assert rel_err(g1, g0) <= 1e-13


def test_culled_sknr_and_top_modes_match_dense():
    """Culled Newton derivative pass (DMMA, r from a culled row LSE) and culled
    top_modes operator passes (normalised by the anchor's own transforms)."""
    r = np.random.default_rng(11)
    n = m = 8192
    x = np.asfortranarray(r.uniform(0, 1, (n, 2)))
    y = np.asfortranarray(r.uniform(0, 1, (m, 2)))
    a = np.full(n, 1.0 / n)
    b = np.full(m, 1.0 / m)
    eps, ell = 2e-3, 12
    pd = sk.PointProblem(x, y, a, b, eps)
    pc = sk.PointProblem(x, y, a, b, eps)
    pc.set_culling(60.0)
    wd = sk.solve(pd.with_epsilon(2 * eps), tol=1e-9, trace=False)
    bd = sk.top_modes(pd.with_epsilon(2 * eps), wd.f, wd.g, ell)
    bc = sk.top_modes(pc.with_epsilon(2 * eps), wd.f, wd.g, ell)
    assert rel_err(bc.rhos, bd.rhos) <= 1e-9
    assert sk.projector_distance(bc, bd) <= 1e-6
    rd = sk.solve(pd, tol=1e-9, ell=ell, basis=bd, init=(wd.f, wd.g))
    rc = sk.solve(pc, tol=1e-9, ell=ell, basis=bd, init=(wd.f, wd.g))
    assert rd.converged and rc.converged
    assert abs(rc.iterations - rd.iterations) <= 1
    assert rel_err(rc.f, rd.f) <= 2e-8  # accept decisions at the rounding level (TOL_POT_NEWTON)


def test_culled_anneal_and_batch_match_dense():
    """Culling inside anneal (epsilon changes between stages, bounds recomputed per pass)
    and inside solve_batch (per-problem work queues)."""
    inst = G.config("C2", n=4096, m=4096)
    mk = lambda: sk.PointProblem(inst.x, inst.y, inst.alpha, inst.beta, inst.epsilons[0], inst.cost_scale)
    pd, pc = mk(), mk()
    pc.set_culling(60.0)
    eps = list(inst.epsilons[:5])
    sd = sk.anneal(pd, eps, warm="potentials", ell=0)
    sc = sk.anneal(pc, eps, warm="potentials", ell=0)
    for a, c in zip(sd, sc):
        assert a.iterations == c.iterations and a.converged and c.converged
        assert rel_err(c.f, a.f) <= 1e-12
    probs = [mk() for _ in range(3)]
    for p in probs:
        p.set_epsilon(inst.epsilons[3])
        p.set_culling(60.0)
    rb = sk.solve_batch(probs, tol=1e-9)
    ref = sk.solve(pd.with_epsilon(inst.epsilons[3]), tol=1e-9)
    for r in rb:
        assert r.iterations == ref.iterations and rel_err(r.f, ref.f) <= 1e-12


@pytest.mark.parametrize("world", [2, 3, 8])
def test_sharded_path_across_R_matches_unsharded(world):
    """SURVEY 8(e) parity across R on one GPU: R emulated ranks (in-process collectives,
    one host thread per rank) run the row-sharded SK and SK-NR solves and top_modes;
    identical iteration counts and potentials within 1e-12 of the unsharded runs."""
    inst = G.config("C1", n=601, m=433)  # ragged row blocks for every R
    a = np.full(601, 1 / 601)
    b = np.full(433, 1 / 433)
    mk = lambda: sk.PointProblem(inst.x, inst.y, a, b, inst.epsilon)
    ref_sk = sk.solve(mk(), tol=1e-9)
    warm = sk.solve(mk().with_epsilon(inst.basis_eps), tol=1e-10)
    basis = sk.top_modes(mk().with_epsilon(inst.basis_eps), warm.f, warm.g, 6)
    ref_nr = sk.solve(mk(), tol=1e-9, ell=6, basis=basis, init=(warm.f, warm.g), accept="stable")
    ref_tm = sk.top_modes(mk(), ref_sk.f, ref_sk.g, 6)
    sched = [0.05, 0.025, 0.0125]
    ref_an = sk.anneal(mk(), sched, warm="spectral", ell=4, accept="stable")
    out = sk.run_emulated_shards(mk, world, lambda p: (
        sk.solve(p, tol=1e-9),
        sk.solve(p, tol=1e-9, ell=6, basis=basis, init=(warm.f, warm.g), accept="stable"),
        sk.top_modes(p, ref_sk.f, ref_sk.g, 6),
        sk.anneal(p, sched, warm="spectral", ell=4, accept="stable")))
    for _, _, _, an in out:
        assert [s.iterations for s in an] == [s.iterations for s in ref_an]
        assert [[t.newton_accepted for t in s.trace] for s in an] == \
            [[t.newton_accepted for t in s.trace] for s in ref_an]
        # stages >= 1 run on a basis each side computed (sharded vs unsharded top_modes,
        # residual tol 1e-8): the Newton directions agree to that resolution only
        assert all(rel_err(s.f, q.f) <= TOL_ANNEAL_BASIS for s, q in zip(an, ref_an))
    out = [o[:3] for o in out]
    for r_sk, r_nr, tm in out:
        assert r_sk.iterations == ref_sk.iterations
        assert rel_err(r_sk.f, ref_sk.f) <= 1e-12 and rel_err(r_sk.g, ref_sk.g) <= 1e-12
        assert r_nr.iterations == ref_nr.iterations
        assert [t.newton_accepted for t in r_nr.trace] == [t.newton_accepted for t in ref_nr.trace]
        assert rel_err(r_nr.f, ref_nr.f) <= TOL_NR
        assert rel_err(tm.rhos, ref_tm.rhos) <= 1e-8
        assert sk.projector_distance(tm, ref_tm) <= 1e-6
    # every rank returns the same full-length potentials
    for r_sk, r_nr, _ in out[1:]:
        assert np.array_equal(r_sk.f, out[0][0].f) and np.array_equal(r_nr.g, out[0][1].g)


TOL_NR = 1e-9  # stable accept test: identical decisions across R


def test_coupling_sharded_rows():
    """coupling_from on R = 3 emulated row shards (core.cpp:84-103): each rank returns its
    own rows of the plan, bitwise equal to the unsharded plan's rows; global row ranges
    outside the rank's block are rejected."""
    inst = G.config("C1", n=301, m=233)
    mk = lambda: sk.PointProblem(inst.x, inst.y, inst.alpha[:301] / inst.alpha[:301].sum(),
                                 inst.beta[:233] / inst.beta[:233].sum(), inst.epsilon)
    ref = sk.solve(mk(), tol=1e-9)
    full = sk.coupling(mk(), ref.f, ref.g)

    def per_rank(p):
        b, e = p._rows
        blk = sk.coupling(p, ref.f, ref.g)
        part = sk.coupling_rows(p, ref.f, ref.g, b + 1, e)
        with pytest.raises(ValueError, match="outside this rank"):
            sk.coupling_rows(p, ref.f, ref.g, max(0, b - 1), e) if b > 0 else \
                sk.coupling_rows(p, ref.f, ref.g, b, e + 1)
        return b, e, blk, part

    for b, e, blk, part in sk.run_emulated_shards(mk, 3, per_rank):
        assert np.array_equal(blk, full[b:e]) and np.array_equal(part, full[b + 1:e])


@pytest.mark.parametrize("world", [1, 3])
def test_householder_fallback_sharded(world, monkeypatch):
    """orthonormalize_deflated's Householder path (spectral.cpp:116-117) forced on every
    round (SKNR_FORCE_HOUSEHOLDER=1), unsharded and on R = 3 emulated row shards (each
    rank gathers the n x k block, runs the same device QR and keeps its rows): the same
    modes as the CholeskyQR3 default."""
    inst = G.config("C1", n=601, m=433)
    a = np.full(601, 1 / 601)
    b = np.full(433, 1 / 433)
    mk = lambda: sk.PointProblem(inst.x, inst.y, a, b, inst.epsilon)
    ref_sk = sk.solve(mk(), tol=1e-9)
    ref_tm = sk.top_modes(mk(), ref_sk.f, ref_sk.g, 6)
    monkeypatch.setenv("SKNR_FORCE_HOUSEHOLDER", "1")
    if world == 1:
        out = [sk.top_modes(mk(), ref_sk.f, ref_sk.g, 6)]
    else:
        out = sk.run_emulated_shards(mk, world, lambda p: sk.top_modes(p, ref_sk.f, ref_sk.g, 6))
    for tm in out:
        assert rel_err(tm.rhos, ref_tm.rhos) <= 1e-8
        assert sk.projector_distance(tm, ref_tm) <= 1e-6
    for tm in out[1:]:
        assert np.array_equal(tm.vectors, out[0].vectors)
TOL_ANNEAL_BASIS = 2e-8


@pytest.mark.parametrize("method,degree", [("chebyshev", 8), ("lanczos", 4)])
def test_sharded_opt_in_basis_methods_match_unsharded(method, degree):
    """The opt-in basis methods bench.py runs on row-sharded C4 under torchrun: the
    Chebyshev-filtered subspace iteration and block Lanczos on R = 3 emulated ranks
    (ragged rows) give the unsharded rhos to 1e-8 and the same subspace."""
    inst = G.config("C1", n=601, m=433)
    a = np.full(601, 1 / 601)
    b = np.full(433, 1 / 433)
    mk = lambda: sk.PointProblem(inst.x, inst.y, a, b, inst.basis_eps)
    warm = sk.solve(mk(), tol=1e-10)
    ref = sk.top_modes(mk(), warm.f, warm.g, 6, method=method, degree=degree)
    out = sk.run_emulated_shards(mk, 3, lambda p: sk.top_modes(p, warm.f, warm.g, 6, method=method,
                                                               degree=degree))
    for tm in out:
        assert rel_err(tm.rhos, ref.rhos) <= 1e-8
        assert sk.projector_distance(tm, ref) <= 1e-6
        assert np.array_equal(tm.vectors, out[0].vectors)


def test_culled_sharded_sk_matches_dense_unsharded():
    """Culling on row-sharded handles (each rank culls its own rows against the global
    LSE bound), R = 4 emulated ranks."""
    c = G.config("C4", n=8192, m=8192)
    mk = lambda: sk.PointProblem(c.x, c.y, c.alpha, c.beta, 2e-3)
    ref = sk.solve(mk(), tol=1e-9)

    def run(p):
        p.set_culling(60.0)
        return sk.solve(p, tol=1e-9)

    out = sk.run_emulated_shards(mk, 4, run)
    for r in out:
        assert r.iterations == ref.iterations
        assert rel_err(r.f, ref.f) <= 1e-12 and rel_err(r.g, ref.g) <= 1e-12


def test_solve_small_batch_matches_oracle_and_solve():
    """Whole SK loop in one kernel launch (5 problems: a group of CTAs each): identical
    iteration counts with the CPU oracle and with solve(), potentials within 1e-9."""
    probs, refs = [], []
    for s in range(5):
        inst = G.config("C1", seed=1 + s, n=300 + 40 * s, m=260 + 30 * s)
        a = np.full(inst.n, 1 / inst.n)
        b = np.full(inst.m, 1 / inst.m)
        probs.append((inst.x, inst.y, a, b, inst.epsilon))
        refs.append(O.solve(O.Instance(a, b, inst.epsilon, x=inst.x, y=inst.y), tol=1e-9))
    out = sk.solve_small_batch(probs, tol=1e-9)
    for (x, y, a, b, e), r, ref in zip(probs, out, refs):
        assert r.converged and r.iterations == ref["iterations"]
        assert rel_err(r.f, ref["f"]) <= 1e-9 and rel_err(r.g, ref["g"]) <= 1e-9
        one = sk.solve(sk.PointProblem(x, y, a, b, e), tol=1e-9)
        assert one.iterations == r.iterations
    with pytest.raises(ValueError, match="n, m <= 8192"):
        x = np.random.default_rng(0).uniform(0, 1, (9000, 2))
        sk.solve_small_batch([(x, x, np.full(9000, 1 / 9000), np.full(9000, 1 / 9000), 0.1)])


def test_solve_small_batch_cta_groups():
    """A lone problem is spread over a cooperative group of CTAs (group barriers, two per
    iteration); a full batch runs one CTA per problem. Both give solve()'s iteration
    count, and the two layouts agree to rounding."""
    inst = G.config("C1")
    a = np.full(inst.n, 1 / inst.n)
    b = np.full(inst.m, 1 / inst.m)
    tup = (inst.x, inst.y, a, b, inst.epsilon)
    ref = sk.solve(sk.PointProblem(*tup), tol=1e-9)
    one = sk.solve_small_batch([tup], tol=1e-9)[0]
    many = sk.solve_small_batch([tup] * 300, tol=1e-9)
    assert one.converged and one.iterations == ref.iterations
    assert rel_err(one.f, ref.f) <= 1e-9 and rel_err(one.g, ref.g) <= 1e-9
    for r in (many[0], many[150], many[299]):
        assert r.iterations == one.iterations
        assert rel_err(r.f, one.f) <= 1e-12 and rel_err(r.g, one.g) <= 1e-12
    assert np.array_equal(many[0].f, many[299].f)
    # C2-sized single problem: 4096 x 4096 on (up to) every SM
    c2 = G.config("C2")
    p2 = (c2.x, c2.y, c2.alpha, c2.beta, 0.02, c2.cost_scale)
    r2 = sk.solve_small_batch([p2], tol=1e-9)[0]
    s2 = sk.solve(sk.PointProblem(c2.x, c2.y, c2.alpha, c2.beta, 0.02, c2.cost_scale), tol=1e-9)
    assert r2.converged and r2.iterations == s2.iterations
    assert rel_err(r2.f, s2.f) <= 1e-9 and rel_err(r2.g, s2.g) <= 1e-9
    # ragged sizes and d = 3 in one batch of two (two groups side by side)
    rng = np.random.default_rng(7)
    ps = []
    for n_, m_ in ((700, 1300), (1901, 33)):
        ps.append((rng.uniform(0, 1, (n_, 3)), rng.normal(size=(m_, 3)), np.full(n_, 1 / n_),
                   np.full(m_, 1 / m_), 0.05))
    outs = sk.solve_small_batch(ps, tol=1e-9)
    for p, r in zip(ps, outs):
        s_ = sk.solve(sk.PointProblem(*p), tol=1e-9)
        assert r.converged and r.iterations == s_.iterations
        assert rel_err(r.f, s_.f) <= 1e-9
