"""Desk-scale harness functions of the reference (namespace sknr::harness and the
dense diagnostics of objective.hpp), built on the GPU primitives of this package.

These are ground-truth / reporting tools, not the solve path: the n x n dense
Hessian and its Cholesky factor are small host matrices (n <= dense_limit),
every O(n m) pass still runs on the device through the C ABI.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import (Problem, _check, _ptr, coupling, ctransform_of_f, ctransform_of_g, gauge_normalized, lib,
               marginal_error, plan_marginals, semi_dual_gradient, semi_dual_value)


def full_semi_dual_hessian(problem: Problem, f, dense_limit: int = 2000) -> np.ndarray:
    """Dense n x n semi-dual Hessian -(1/eps)(diag(r) - P~ diag(b) P~^T), symmetrised
    (objective.cpp:150-171): the plan P~_ij b_j and the O(n^2 m) product are computed on
    the device (sknr_full_semi_dual_hessian); the n x n result comes back to the host."""
    if problem.n > dense_limit:
        raise ValueError("full_semi_dual_hessian: dense Hessian too large")
    f = np.ascontiguousarray(f, dtype=np.float64)
    out = np.empty((problem.n, problem.n), order="F")
    _check(lib().sknr_full_semi_dual_hessian(problem.handle, _ptr(f), int(dense_limit), _ptr(out)))
    return out


@dataclass
class OracleSolution:
    """OracleSolution (harness/oracle.hpp:11-15)."""

    f: np.ndarray
    g: np.ndarray
    plan: np.ndarray
    residual: float

    def __getitem__(self, key):  # dict access like the pybind `oracle_solve` (bindings.cpp:180-191)
        return getattr(self, key)


def _residual(problem: Problem, f, g) -> float:
    return plan_marginals(problem, f, g)[2]


def oracle_solve(problem: Problem, target_residual: float = 1e-13) -> OracleSolution:
    """Ground-truth solve (oracle.cpp:21-90): batches of 50 plain Sinkhorn sweeps
    (each followed by the alpha-gauge), then a damped full-space Newton polish on
    the semi-dual with the gauge direction removed by the rank-one shift
    mu 11^T, mu = 1/(eps n); repeated until the L2 marginal residual is below
    target. Desk scale only (n*m <= 1e6)."""
    n, m = problem.n, problem.m
    if n * m > 1_000_000:
        raise ValueError("oracle_solve: instance above desk scale (n*m > 1e6)")
    alpha = problem.alpha
    f, g = np.zeros(n), np.zeros(m)
    residual = _residual(problem, f, g)
    k_max_sk, k_batch = 10_000_000, 50
    sk_done = 0

    def newton_polish(f, g, residual):
        for _ in range(60):
            if not residual > target_residual:
                break
            hess = full_semi_dual_hessian(problem, f)
            mu = 1.0 / (problem.epsilon * n)
            shifted = -hess + mu * np.ones((n, n))
            try:
                L = np.linalg.cholesky(shifted)
            except np.linalg.LinAlgError:
                return f, g, residual
            grad = semi_dual_gradient(problem, f)
            delta = np.linalg.solve(L.T, np.linalg.solve(L, grad))
            value = semi_dual_value(problem, f)
            step, improved = 1.0, False
            for _ in range(40):
                cand = f + step * delta
                if semi_dual_value(problem, cand) > value:
                    f, improved = cand, True
                    break
                step *= 0.5
            if not improved:
                return f, g, residual
            g = ctransform_of_f(problem, f)
            residual = _residual(problem, f, g)
        return f, g, residual

    while residual > target_residual and sk_done < k_max_sk:
        for _ in range(k_batch):
            if sk_done >= k_max_sk:
                break
            g = ctransform_of_f(problem, f)
            f = ctransform_of_g(problem, g)
            c = float(alpha @ f)
            f = f - c
            g = g + c
            sk_done += 1
        residual = _residual(problem, f, g)
        if residual <= target_residual:
            break
        f, g, residual = newton_polish(f, g, residual)

    if residual > 10.0 * target_residual:
        raise RuntimeError(f"oracle_solve: no convergence, residual {residual}")
    f, g = gauge_normalized(problem, f, g)
    plan = coupling(problem, f, g)
    return OracleSolution(f, g, plan, marginal_error(problem, plan))


__all__ = ["OracleSolution", "full_semi_dual_hessian", "oracle_solve"]
