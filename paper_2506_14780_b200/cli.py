"""Command-line front end mirroring the reference `sknr` CLI (proj/tools/main.cpp),
running every solve on the GPU.

    python -m paper_2506_14780_b200 solve    --points SRC TGT --epsilon E [--ell L --basis-from E'] --out DIR
    python -m paper_2506_14780_b200 spectrum --cost C.csv --epsilons 0.1,0.05 --k 10 [--vectors] --out DIR
    python -m paper_2506_14780_b200 anneal   --synthetic gauss2d --schedule 0.1,0.05 --warm spectral --out DIR

Instances: exactly one of --synthetic (gauss2d | two_moons | annulus_square),
--points (source and target CSVs; squared-Euclidean cost evaluated on the fly,
main.cpp:73-87 would build it dense) or --cost (with optional --alpha/--beta).
Exit codes (main.cpp:3-5): 0 success (converged), 1 input error, 2 max_iter
reached, 3 eigensolver non-convergence. The reference's `experiment`
subcommand (harness experiment configs) is not provided.
"""
from __future__ import annotations

import argparse
import os
import sys

import numpy as np

from . import (EigensolverError, PointProblem, Problem, anneal, solve, spectrum, top_modes)
from . import generators as G
from . import io as sio
from .harness import oracle_solve


def _add_instance_flags(p: argparse.ArgumentParser) -> None:
    p.add_argument("--synthetic", default="", help="Named generator: gauss2d | two_moons | annulus_square")
    p.add_argument("--points", nargs=2, metavar=("SRC", "TGT"), default=None,
                   help="Source and target point-cloud CSVs (squared Euclidean cost)")
    p.add_argument("--cost", default="", help="Cost matrix CSV")
    p.add_argument("--alpha", default="", help="Source weights CSV (with --cost)")
    p.add_argument("--beta", default="", help="Target weights CSV (with --cost)")
    p.add_argument("--seed", type=int, default=1, help="Generator seed (synthetic instances)")
    p.add_argument("--n", type=int, default=200, help="Source size (synthetic instances)")
    p.add_argument("--m", type=int, default=400, help="Target size (synthetic instances)")
    p.add_argument("--noise", type=float, default=0.05, help="two_moons noise level")
    p.add_argument("--r-in", type=float, default=0.5, help="annulus inner radius")
    p.add_argument("--r-out", type=float, default=1.0, help="annulus outer radius")
    p.add_argument("--side", type=float, default=2.0, help="square side length")


def load_instance(a, epsilon: float) -> Problem:
    """load_instance (main.cpp:57-112)."""
    sources = int(bool(a.synthetic)) + int(a.points is not None) + int(bool(a.cost))
    if sources != 1:
        raise ValueError("exactly one of --synthetic, --points, --cost is required")
    if a.synthetic:
        x, wa, y, wb = G.make_instance(a.synthetic, a.n, a.m, a.seed, a.noise, a.r_in, a.r_out, a.side)
        return PointProblem(x, y, wa, wb, epsilon)
    if a.points is not None:
        xs, wa, ren_a = sio.read_point_cloud(a.points[0])
        yt, wb, ren_b = sio.read_point_cloud(a.points[1])
        if ren_a:
            print(f"warning: {a.points[0]}: weights renormalized to sum to 1", file=sys.stderr)
        if ren_b:
            print(f"warning: {a.points[1]}: weights renormalized to sum to 1", file=sys.stderr)
        if xs.shape[1] != yt.shape[1]:
            raise ValueError("sq_euclidean_cost: dimension mismatch")
        return PointProblem(xs, yt, wa, wb, epsilon)
    cost = sio.read_csv_matrix(a.cost)
    wa = sio.read_csv_vector(a.alpha) if a.alpha else np.full(cost.shape[0], 1.0 / cost.shape[0])
    wb = sio.read_csv_vector(a.beta) if a.beta else np.full(cost.shape[1], 1.0 / cost.shape[1])
    for w, name in ((wa, "alpha"), (wb, "beta")):
        total = float(np.sum(w))
        if abs(total - 1.0) > 1e-9:
            print(f"warning: {name}: weights renormalized to sum to 1", file=sys.stderr)
            w /= total
    return Problem(cost, wa, wb, epsilon)


def cmd_solve(a) -> int:
    """cmd_solve (main.cpp:120-157). Opt-in additions (point clouds only, not in the
    reference CLI): --cull T (skip terms below e^-T), --warm-fp32 (the --basis-from warm
    solve with fp32 LSE passes), --basis-method (chebyshev / lanczos top_modes)."""
    problem = load_instance(a, a.epsilon)
    if (a.cull or a.warm_fp32) and not isinstance(problem, PointProblem):
        raise ValueError("--cull / --warm-fp32 need a point-cloud instance (--points or --synthetic)")
    if a.cull:
        problem.set_culling(a.cull)
    basis, init = None, None
    if a.ell > 0:
        warm_eps = a.basis_from if a.basis_from is not None else a.epsilon
        warm_problem = problem.with_epsilon(warm_eps)
        if a.warm_fp32:
            warm_problem.set_precision(32)
        warm = solve(warm_problem, tol=a.tol, max_iter=a.max_iter, ell=0, trace=not a.no_trace)
        if a.warm_fp32:
            warm_problem.set_precision(64)
        degree = 12 if a.basis_method == "lanczos" else 8
        basis = top_modes(warm_problem, warm.f, warm.g, a.ell, method=a.basis_method, degree=degree)
        if a.basis_from is not None:
            init = (warm.f, warm.g)
    result = solve(problem, tol=a.tol, max_iter=a.max_iter, ell=a.ell, basis=basis, init=init,
                   trace=not a.no_trace)
    os.makedirs(a.out, exist_ok=True)
    sio.write_potentials_csv(os.path.join(a.out, "potentials.csv"), result.f, result.g)
    marginal = sio.write_coupling_csv(os.path.join(a.out, "coupling.csv"), problem, result.f, result.g)
    if not a.no_trace:
        sio.write_trace_csv(os.path.join(a.out, "trace.csv"), result.trace)
    print(f"converged={'true' if result.converged else 'false'} iters={result.iterations} "
          f"marginal_error={marginal:.17e}")
    return 0 if result.converged else 2


def cmd_spectrum(a) -> int:
    """cmd_spectrum (main.cpp:159-178): anchor = oracle_solve(problem, 1e-12)."""
    eps_list = [float(e) for e in a.epsilons.split(",") if e]
    if not eps_list:
        raise ValueError("--epsilons is required")
    os.makedirs(a.out, exist_ok=True)
    for idx, eps in enumerate(eps_list):
        problem = load_instance(a, eps)
        anchor = oracle_solve(problem, 1e-12)
        rep = spectrum(problem, anchor.f, anchor.g, a.k, a.vectors)
        name = "spectrum_%03d.json" % idx
        sio.write_spectrum_json(os.path.join(a.out, name), rep, a.k)
        print(f"epsilon={eps:.17g} rho_1={rep['rho'][0]:.17g} file={name}")
    return 0


def cmd_anneal(a) -> int:
    """cmd_anneal (main.cpp:180-218)."""
    schedule = [float(e) for e in a.schedule.split(",") if e]
    if not schedule:
        raise ValueError("--schedule is required")
    if a.warm not in ("none", "potentials", "spectral"):
        raise ValueError("--warm must be none, potentials or spectral")
    problem = load_instance(a, schedule[0])
    stages = anneal(problem, schedule, warm=a.warm, ell=a.ell, refresh_basis=a.refresh_basis, tol=a.tol,
                    max_iter=a.max_iter)
    os.makedirs(a.out, exist_ok=True)
    all_conv = True
    for s, st in enumerate(stages):
        sio.write_potentials_csv(os.path.join(a.out, "stage_%02d_potentials.csv" % s), st.f, st.g)
        print(f"stage={s} epsilon={schedule[s]:.17g} converged={'true' if st.converged else 'false'} "
              f"iters={st.iterations}")
        all_conv = all_conv and st.converged
    sio.write_anneal_csv(os.path.join(a.out, "anneal_trace.csv"), schedule, stages)
    return 0 if all_conv else 2


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="sknr_b200",
                                 description="sknr: accelerated Sinkhorn solver for entropic optimal transport")
    sub = ap.add_subparsers(dest="cmd", required=True)
    s = sub.add_parser("solve", help="Run SK / SK-NR on one instance")
    _add_instance_flags(s)
    s.add_argument("--epsilon", type=float, required=True, help="Regularization")
    s.add_argument("--tol", type=float, default=1e-9, help="Marginal-error tolerance omega")
    s.add_argument("--max-iter", type=int, default=100000, help="Iteration cap")
    s.add_argument("--ell", type=int, default=0, help="Newton subspace dimension")
    s.add_argument("--basis-from", type=float, default=None,
                   help="Build the basis (and warm start) from the solution at this epsilon")
    s.add_argument("--out", default=".", help="Output directory")
    s.add_argument("--no-trace", action="store_true", help="Skip the per-iteration trace file")
    s.add_argument("--cull", type=float, default=0.0,
                   help="Opt-in: skip LSE terms below e^-T of their output's total (point clouds, T >= 40)")
    s.add_argument("--warm-fp32", action="store_true",
                   help="Opt-in: run the --basis-from warm solve with fp32 LSE passes (point clouds)")
    s.add_argument("--basis-method", choices=["subspace", "chebyshev", "lanczos"], default="subspace",
                   help="top_modes method (subspace = the reference's)")
    s.set_defaults(fn=cmd_solve)
    p = sub.add_parser("spectrum", help="Eigen-structure reports across epsilons")
    _add_instance_flags(p)
    p.add_argument("--epsilons", required=True, help="Comma list of epsilons")
    p.add_argument("--k", type=int, default=10, help="Number of modes")
    p.add_argument("--vectors", action="store_true", help="Export eigenvectors")
    p.add_argument("--out", default=".", help="Output directory")
    p.set_defaults(fn=cmd_spectrum)
    n = sub.add_parser("anneal", help="Epsilon-annealing with warm starts")
    _add_instance_flags(n)
    n.add_argument("--schedule", required=True, help="Decreasing epsilon list")
    n.add_argument("--warm", default="none", help="none | potentials | spectral")
    n.add_argument("--ell", type=int, default=8, help="Newton subspace dimension")
    n.add_argument("--refresh-basis", action="store_true", help="Rebuild the basis every stage")
    n.add_argument("--tol", type=float, default=1e-9, help="Marginal-error tolerance omega")
    n.add_argument("--max-iter", type=int, default=100000, help="Iteration cap")
    n.add_argument("--out", default=".", help="Output directory")
    n.set_defaults(fn=cmd_anneal)
    return ap


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    try:
        return args.fn(args)
    except EigensolverError as e:
        print(f"error: {e}", file=sys.stderr)
        return 3
    except Exception as e:  # std::exception -> 1 (main.cpp:335-338)
        print(f"error: {e}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
