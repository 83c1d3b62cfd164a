"""B200-native SK-NR(ell) core (arXiv 2506.14780) -- Python mirror of the
reference's `sknr` module (/root/reference/proj/python/bindings.cpp:35-215).

Every compute call goes through libsknr_b200.so (C ABI, include/sknr_gpu.h) on
an sm_100a device. There is no CPU fallback: if the library is missing or no
CUDA device is usable, calls raise RuntimeError.

Names, argument meaning and error behaviour follow the reference bindings:
`Problem(cost, alpha, beta, epsilon)`, `solve(problem, tol, max_iter, ell,
basis, init, trace)`, `top_modes(problem, f, g, ell, tol, max_power_iters)`,
`anneal(problem, epsilons, warm, ell, refresh_basis, tol, max_iter)`, the
transforms and objective helpers. `PointProblem` is the on-the-fly cost variant
(C_ij = cost_scale * ||x_i - y_j||^2 never stored) the north star adds.
Invalid arguments raise ValueError (pybind11 maps std::invalid_argument to
ValueError), EigensolverError carries best_residual.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

__version__ = "0.1.0"

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.environ.get("SKNR_B200_LIB", os.path.join(_HERE, "libsknr_b200.so"))
_lib = None

SKNR_OK, SKNR_EINVAL, SKNR_EEIGEN, SKNR_ECUDA, SKNR_ENCCL, SKNR_ERUNTIME = 0, 1, 2, 3, 4, 5


class EigensolverError(RuntimeError):
    """top_modes did not reach its residual target (spectral.hpp:60-68)."""

    def __init__(self, msg: str, best_residual: float):
        super().__init__(msg)
        self.best_residual = best_residual


class _Config(ctypes.Structure):
    _fields_ = [
        ("tol_omega", ctypes.c_double),
        ("max_iter", ctypes.c_int64),
        ("ell", ctypes.c_int64),
        ("newton_enabled", ctypes.c_int32),
        ("trace_enabled", ctypes.c_int32),
        ("exact_marginals", ctypes.c_int32),
        ("accept_test", ctypes.c_int32),
    ]


class _Record(ctypes.Structure):
    _fields_ = [
        ("index", ctypes.c_int64),
        ("marginal_error", ctypes.c_double),
        ("marginal_error_inf", ctypes.c_double),
        ("semi_dual_value", ctypes.c_double),
        ("newton_attempted", ctypes.c_int32),
        ("newton_accepted", ctypes.c_int32),
        ("wall_time_ms", ctypes.c_double),
    ]


_D = ctypes.POINTER(ctypes.c_double)
_I64 = ctypes.c_int64
_P = ctypes.c_void_p

# name -> argtypes (all return int status unless listed in _RET)
_SIGS = {
    "sknr_last_error": [],
    "sknr_last_best_residual": [],
    "sknr_version": [ctypes.c_char_p, ctypes.c_int],
    "sknr_kernel_launch_count": [],
    "sknr_problem_create_dense": [_D, _I64, _I64, _D, _D, ctypes.c_double, ctypes.POINTER(_P)],
    "sknr_problem_create_points": [_D, _D, _I64, _I64, _I64, ctypes.c_double, _D, _D,
                                   ctypes.c_double, ctypes.POINTER(_P)],
    "sknr_problem_create_points_ex": [_D, _D, _I64, _I64, _I64, ctypes.c_double, _D, _D,
                                      ctypes.c_double, ctypes.c_int, ctypes.POINTER(_P)],
    "sknr_problem_set_epsilon": [_P, ctypes.c_double],
    "sknr_problem_info": [_P, ctypes.POINTER(_I64), ctypes.POINTER(_I64), ctypes.POINTER(_I64),
                          _D, ctypes.POINTER(ctypes.c_int)],
    "sknr_problem_destroy": [_P],
    "sknr_problem_set_culling": [_P, ctypes.c_double],
    "sknr_problem_set_precision": [_P, ctypes.c_int],
    "sknr_ctransform_of_f": [_P, _D, _D],
    "sknr_ctransform_of_g": [_P, _D, _D],
    "sknr_plan_marginals": [_P, _D, _D, _D, _D, _D, _D],
    "sknr_coupling": [_P, _D, _D, _D],
    "sknr_coupling_rows": [_P, _D, _D, _I64, _I64, _D],
    "sknr_solve_small_batch": [_I64, _I64, ctypes.POINTER(_I64), ctypes.POINTER(_I64), ctypes.POINTER(_D),
                               ctypes.POINTER(_D), ctypes.POINTER(_D), ctypes.POINTER(_D), _D, _D, ctypes.c_double,
                               _I64, ctypes.POINTER(_D), ctypes.POINTER(_D), ctypes.POINTER(_I64),
                               ctypes.POINTER(ctypes.c_int)],
    "sknr_solve_batch": [ctypes.POINTER(_P), _I64, ctypes.POINTER(_Config), ctypes.POINTER(_D), _I64,
                         ctypes.POINTER(_D), ctypes.POINTER(_D), ctypes.POINTER(_D), ctypes.POINTER(_D),
                         ctypes.POINTER(_I64), ctypes.POINTER(ctypes.c_int)],
    "sknr_apply_R": [_P, _D, _D, _D, _D],
    "sknr_apply_Rt": [_P, _D, _D, _D, _D],
    "sknr_dual_value": [_P, _D, _D, _D],
    "sknr_semi_dual_hessian_quadform": [_P, _D, _D, _D],
    "sknr_full_semi_dual_hessian": [_P, _D, _I64, _D],
    "sknr_newton_step": [_P, _D, _D, _I64, _D, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int)],
    "sknr_newton_step_ex": [_P, _D, _D, _I64, ctypes.c_int, _D, ctypes.POINTER(ctypes.c_int),
                            ctypes.POINTER(ctypes.c_int)],
    "sknr_last_trace": [_P, ctypes.POINTER(_Record), _I64, ctypes.POINTER(_I64)],
    "sknr_spectrum_report": [_P, _D, _D, _I64, ctypes.c_int, ctypes.c_double, _I64, _D, _D, _D, _D, _D],
    "sknr_projector_distance": [_I64, _I64, _D, _D, _D],
    "sknr_semi_dual_value": [_P, _D, _D],
    "sknr_restricted_derivatives": [_P, _D, _D, _D, _I64, _D, _D],
    "sknr_apply_sym_block": [_P, _D, _D, _D, _I64, _D],
    "sknr_apply_sym_t_block": [_P, _D, _D, _D, _I64, _D],
    "sknr_top_modes": [_P, _D, _D, _I64, ctypes.c_double, _I64, _D, _D, _D,
                       ctypes.POINTER(_I64)],
    "sknr_top_modes_ex": [_P, _D, _D, _I64, ctypes.c_double, _I64, ctypes.c_int, ctypes.c_int, _D, _D, _D,
                          ctypes.POINTER(_I64)],
    "sknr_config_default": [ctypes.POINTER(_Config)],
    "sknr_solve": [_P, ctypes.POINTER(_Config), _D, _I64, _D, _D, _D, _D, ctypes.POINTER(_I64),
                   ctypes.POINTER(ctypes.c_int), ctypes.POINTER(_Record), _I64,
                   ctypes.POINTER(_I64)],
    "sknr_anneal": [_P, _D, _I64, ctypes.c_int, ctypes.c_int, ctypes.POINTER(_Config), _D, _D,
                    ctypes.POINTER(_I64), ctypes.POINTER(ctypes.c_int), ctypes.POINTER(_Record),
                    _I64, ctypes.POINTER(_I64), ctypes.POINTER(_I64)],
    "sknr_bench_pass": [_P, ctypes.c_int, _I64, ctypes.c_int, _D, _D],
    "sknr_bench_iterations": [_P, ctypes.POINTER(_Config), _D, _I64, _I64, _I64, ctypes.c_int, _D,
                              ctypes.POINTER(_I64)],
    "sknr_bench_fp64_peak": [_D, _D],
    "sknr_bench_mufu_peak": [_D, _D],
    "sknr_tune_variant": [_P, ctypes.c_int, ctypes.c_int, _D],
    "sknr_debug_counters": [_P, ctypes.POINTER(_I64)],
    "sknr_set_tensor_block_pass": [ctypes.c_int],
    "sknr_get_tensor_block_pass": [],
    "sknr_probe_i8_mma": [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_void_p],
    "sknr_comm_unique_id": [ctypes.c_void_p],
    "sknr_comm_init": [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_int],
    "sknr_comm_destroy": [],
    "sknr_comm_init_emulated": [ctypes.c_int],
    "sknr_problem_shard": [_P, _I64, _I64],
    "sknr_comm_stats": [ctypes.POINTER(_I64), ctypes.POINTER(_I64), ctypes.c_int],
}
_RET = {
    "sknr_last_error": ctypes.c_char_p,
    "sknr_last_best_residual": ctypes.c_double,
    "sknr_kernel_launch_count": ctypes.c_int64,
    "sknr_config_default": None,
}


def library_path() -> str:
    return _LIB_PATH


def lib():
    """Load libsknr_b200.so (raises if it was not built -- no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH):
        raise RuntimeError(
            f"sknr_b200: native library {_LIB_PATH} is missing; run "
            "`python -c 'import __graft_entry__ as g; g.build()'` (there is no CPU fallback)")
    handle = ctypes.CDLL(_LIB_PATH)
    for name, args in _SIGS.items():
        fn = getattr(handle, name)
        fn.argtypes = args
        fn.restype = _RET.get(name, ctypes.c_int)
    _lib = handle
    return _lib


def _check(rc: int) -> None:
    if rc == SKNR_OK:
        return
    msg = lib().sknr_last_error().decode()
    if rc == SKNR_EINVAL:
        raise ValueError(msg)
    if rc == SKNR_EEIGEN:
        raise EigensolverError(msg, lib().sknr_last_best_residual())
    raise RuntimeError(msg)


def _vec(x, name="vector") -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(x, dtype=np.float64).reshape(-1))
    return a


def _mat_f(x) -> np.ndarray:
    """Column-major (Fortran) float64 copy, like Eigen::MatrixXd."""
    return np.asfortranarray(np.asarray(x, dtype=np.float64))


def _ptr(a: Optional[np.ndarray]):
    if a is None:
        return None
    return a.ctypes.data_as(_D)


def version() -> str:
    buf = ctypes.create_string_buffer(256)
    _check(lib().sknr_version(buf, 256))
    return buf.value.decode()


def kernel_launch_count() -> int:
    return int(lib().sknr_kernel_launch_count())


# ---------------------------------------------------------------- problems
class Problem:
    """EotProblem (types.hpp:47-69) with a dense n x m cost, resident on the GPU."""

    _kind = 0

    def __init__(self, cost, alpha, beta, epsilon: float):
        cost = _mat_f(cost)
        if cost.ndim != 2:
            raise ValueError("CostMatrix: need a 2-d matrix")
        n, m = cost.shape
        a, b = _vec(alpha), _vec(beta)
        if a.size != n or b.size != m:
            raise ValueError("EotProblem: measure sizes must match cost shape")
        h = _P()
        _check(lib().sknr_problem_create_dense(_ptr(cost), n, m, _ptr(a), _ptr(b), float(epsilon),
                                               ctypes.byref(h)))
        self._init_common(h, n, m, a, b, float(epsilon))
        self._cost = cost

    def _init_common(self, h, n, m, a, b, eps):
        self._h = h
        self._n, self._m = int(n), int(m)
        self._alpha, self._beta = a, b
        self._eps = eps

    @property
    def n(self) -> int:
        return self._n

    @property
    def m(self) -> int:
        return self._m

    @property
    def epsilon(self) -> float:
        return self._eps

    @property
    def alpha(self) -> np.ndarray:
        return self._alpha.copy()

    @property
    def beta(self) -> np.ndarray:
        return self._beta.copy()

    @property
    def cost(self) -> np.ndarray:
        return self._cost

    def with_epsilon(self, epsilon: float) -> "Problem":
        """Same instance at another regularisation (types.hpp:60-62)."""
        return type(self)._clone(self, float(epsilon))

    @classmethod
    def _clone(cls, p: "Problem", eps: float):
        if isinstance(p, PointProblem):
            q = PointProblem(p._x, p._y, p._alpha, p._beta, eps, p._cost_scale, p._cost_mode)
            if getattr(p, "_cull", 0.0) > 0.0:
                q.set_culling(p._cull)
            if getattr(p, "_precision", 64) != 64:
                q.set_precision(p._precision)
            return q
        return Problem(p._cost, p._alpha, p._beta, eps)

    def set_epsilon(self, epsilon: float) -> None:
        """In-place epsilon change (no cost copy, unlike with_epsilon)."""
        _check(lib().sknr_problem_set_epsilon(self._h, float(epsilon)))
        self._eps = float(epsilon)

    @property
    def handle(self):
        return self._h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None:
            _lib.sknr_problem_destroy(h)
            self._h = None


class PointProblem(Problem):
    """On-the-fly squared-Euclidean cost C_ij = cost_scale * ||x_i - y_j||^2
    (sq_euclidean_cost, generators.cpp:94-103) between point clouds x (n x d)
    and y (m x d); the n x m cost is never stored for d <= 4."""

    _kind = 1

    COST_MODES = {"auto": 0, "stored": 1, "onthefly": 2}

    def __init__(self, x, y, alpha, beta, epsilon: float, cost_scale: float = 1.0, cost_mode: str = "auto"):
        """cost_mode: "auto" (d <= 4 in registers; d > 4 stored when 2nm doubles fit in
        HBM, else on the fly), "stored", "onthefly" (d > 4: x.y contraction on FP64
        tensor cores)."""
        if cost_mode not in self.COST_MODES:
            raise ValueError("cost_mode must be auto|stored|onthefly")
        x, y = _mat_f(x), _mat_f(y)
        if x.ndim == 1:
            x = x.reshape(-1, 1, order="F")
        if y.ndim == 1:
            y = y.reshape(-1, 1, order="F")
        if x.shape[1] != y.shape[1]:
            raise ValueError("sq_euclidean_cost: dimension mismatch")
        n, d = x.shape
        m = y.shape[0]
        a, b = _vec(alpha), _vec(beta)
        if a.size != n or b.size != m:
            raise ValueError("EotProblem: measure sizes must match cost shape")
        h = _P()
        _check(lib().sknr_problem_create_points_ex(_ptr(x), _ptr(y), n, m, d, float(cost_scale), _ptr(a),
                                                   _ptr(b), float(epsilon), self.COST_MODES[cost_mode],
                                                   ctypes.byref(h)))
        self._init_common(h, n, m, a, b, float(epsilon))
        self._x, self._y, self._cost_scale = x, y, float(cost_scale)
        self._cost_mode = cost_mode

    def set_culling(self, threshold: float = 60.0) -> None:
        """Opt-in: skip LSE terms provably below e^-threshold of their output's total
        (Morton-ordered group bounds; 0 disables). Not in the reference API."""
        _check(lib().sknr_problem_set_culling(self.handle, float(threshold)))
        self._cull = float(threshold)

    def set_precision(self, bits: int) -> None:
        """Opt-in: bits=32 runs the LSE sum passes with fp32 cell exponents and MUFU exp2
        (accumulation and potentials stay fp64; potentials within ~1e-5 relative of the
        fp64 path); bits=64 (default) is the reference's arithmetic. Not in the reference API."""
        _check(lib().sknr_problem_set_precision(self.handle, int(bits)))
        self._precision = int(bits)

    @property
    def cost(self) -> np.ndarray:
        diff = self._x[:, None, :] - self._y[None, :, :]
        return np.asfortranarray(self._cost_scale * np.einsum("ijk,ijk->ij", diff, diff))

    @property
    def d(self) -> int:
        return self._x.shape[1]

    @property
    def cost_path(self) -> str:
        """Which kernel family evaluates the cost: registers / contraction / stored."""
        kind = ctypes.c_int()
        _check(lib().sknr_problem_info(self.handle, None, None, None, None, ctypes.byref(kind)))
        return {0: "stored", 1: "registers", 2: "contraction"}[kind.value]


# ---------------------------------------------------------------- results
@dataclass
class SpectralBasis:
    """SpectralBasis (spectral.hpp:48-56)."""

    vectors: np.ndarray
    vectors_sym: np.ndarray
    rhos: np.ndarray
    epsilon_built_at: float
    sweeps: int = 0

    @property
    def ell(self) -> int:
        return self.vectors.shape[1]

    @property
    def dim(self) -> int:
        return self.vectors.shape[0]


@dataclass
class IterationRecord:
    index: int
    marginal_error: float
    marginal_error_inf: float
    semi_dual_value: float
    newton_attempted: bool
    newton_accepted: bool
    wall_time_ms: float


@dataclass
class SolveResult:
    f: np.ndarray
    g: np.ndarray
    converged: bool
    iterations: int
    trace: list = field(default_factory=list)
    _problem: Optional[Problem] = None
    _epsilon: Optional[float] = None

    @property
    def plan(self) -> np.ndarray:
        """coupling_from at the returned potentials (solver.cpp:154), materialised on demand."""
        p = self._problem
        if self._epsilon is not None and self._epsilon != p.epsilon:
            p = p.with_epsilon(self._epsilon)
        return coupling(p, self.f, self.g)


def _records(buf, count) -> list:
    return [IterationRecord(int(r.index), r.marginal_error, r.marginal_error_inf, r.semi_dual_value,
                            bool(r.newton_attempted), bool(r.newton_accepted), r.wall_time_ms)
            for r in buf[:count]]


# ---------------------------------------------------------------- core.hpp
def log_sum_exp(values, log_weights) -> float:
    """log sum_i exp(values_i + log_weights_i), max-shifted (core.cpp:9-22).
    Host-side scalar helper of the reference API (not on the O(nm) path)."""
    v, w = _vec(values), _vec(log_weights)
    if v.size == 0 or w.size == 0:
        raise ValueError("log_sum_exp: empty reduction")
    if v.size != w.size:
        raise ValueError("log_sum_exp: length mismatch")
    shift = -np.inf
    for i in range(v.size):
        shift = max(shift, v[i] + w[i])
    total = 0.0
    for i in range(v.size):
        total += np.exp(v[i] + w[i] - shift)
    return float(shift + np.log(total))


def _checked(v, size, what):
    a = _vec(v)
    if a.size != size:
        raise ValueError(f"{what}: length mismatch")
    if not np.all(np.isfinite(a)):
        raise ValueError(f"{what}: entries must be finite")
    return a


def ctransform_of_f(problem: Problem, f) -> np.ndarray:
    f = _checked(f, problem.n, "ctransform_of_f")
    g = np.empty(problem.m)
    _check(lib().sknr_ctransform_of_f(problem.handle, _ptr(f), _ptr(g)))
    return g


def ctransform_of_g(problem: Problem, g) -> np.ndarray:
    g = _checked(g, problem.m, "ctransform_of_g")
    f = np.empty(problem.n)
    _check(lib().sknr_ctransform_of_g(problem.handle, _ptr(g), _ptr(f)))
    return f


def plan_marginals(problem: Problem, f, g):
    """(row, col, gap_l2, gap_inf) of the plan induced by (f, g) (core.cpp:120-150)."""
    f = _checked(f, problem.n, "plan_marginals(f)")
    g = _checked(g, problem.m, "plan_marginals(g)")
    row, col = np.empty(problem.n), np.empty(problem.m)
    l2, inf = ctypes.c_double(), ctypes.c_double()
    _check(lib().sknr_plan_marginals(problem.handle, _ptr(f), _ptr(g), _ptr(row), _ptr(col),
                                     ctypes.byref(l2), ctypes.byref(inf)))
    return row, col, l2.value, inf.value


def coupling(problem: Problem, f, g) -> np.ndarray:
    """coupling_from (core.cpp:84-103); on a row-sharded problem, this rank's rows
    (row_partition) -- each rank materialises its own block of the n x m plan."""
    f = _checked(f, problem.n, "coupling_from(f)")
    g = _checked(g, problem.m, "coupling_from(g)")
    b, e = getattr(problem, "_rows", (0, problem.n))
    plan = np.empty((e - b, problem.m), order="F")
    _check(lib().sknr_coupling(problem.handle, _ptr(f), _ptr(g), _ptr(plan)))
    return plan


def coupling_rows(problem: Problem, f, g, row_begin: int, row_end: int) -> np.ndarray:
    """Rows [row_begin, row_end) of coupling_from's plan (for streaming an n x m plan)."""
    f = _checked(f, problem.n, "coupling_from(f)")
    g = _checked(g, problem.m, "coupling_from(g)")
    rows = int(row_end) - int(row_begin)
    if rows < 0:
        raise ValueError("coupling_rows: row range out of bounds")
    block = np.empty((rows, problem.m), order="F")
    _check(lib().sknr_coupling_rows(problem.handle, _ptr(f), _ptr(g), int(row_begin), int(row_end),
                                    _ptr(block)))
    return block


def marginal_gap(problem: Problem, row, col):
    """(l2, inf) = (||row - alpha||_2 + ||col - beta||_2, ||.||_inf + ||.||_inf) (core.cpp:145-150)."""
    row, col = _vec(row), _vec(col)
    if row.size != problem.n or col.size != problem.m:
        raise ValueError("marginal_gap: length mismatch")
    dr, dc = row - problem._alpha, col - problem._beta
    return (float(np.linalg.norm(dr) + np.linalg.norm(dc)),
            float(np.max(np.abs(dr)) + np.max(np.abs(dc))))


def gauge_normalized(problem: Problem, f, g):
    """(f - c, g + c) with c = alpha . f (core.cpp:152-157)."""
    f, g = _vec(f), _vec(g)
    c = float(problem._alpha @ f)
    return f - c, g + c


def gauge_distance(problem: Problem, a, b) -> float:
    """max |.| between gauge-normalised potential pairs a=(f,g), b=(f,g) (core.cpp:159-165)."""
    fa, ga = gauge_normalized(problem, *a)
    fb, gb = gauge_normalized(problem, *b)
    return float(max(np.max(np.abs(fa - fb)), np.max(np.abs(ga - gb))))


def marginal_error(problem: Problem, plan) -> float:
    """||plan 1 - alpha||_2 + ||plan^T 1 - beta||_2 (core.cpp:105-112)."""
    plan = np.asarray(plan, dtype=np.float64)
    if plan.shape != (problem.n, problem.m):
        raise ValueError("marginal_error: plan shape mismatch")
    return float(np.linalg.norm(plan.sum(axis=1) - problem._alpha) +
                 np.linalg.norm(plan.sum(axis=0) - problem._beta))


def osc_norm(v) -> float:
    v = _vec(v)
    if v.size == 0:
        raise ValueError("osc_norm: empty input")
    return float(v.max() - v.min())


# ---------------------------------------------------------------- objective.hpp
def semi_dual_value(problem: Problem, f) -> float:
    f = _checked(f, problem.n, "ctransform_of_f")
    out = ctypes.c_double()
    _check(lib().sknr_semi_dual_value(problem.handle, _ptr(f), ctypes.byref(out)))
    return out.value


def dual_value(problem: Problem, f, g) -> float:
    """a.f + b.g - eps*expm1(log sum_ij a_i b_j e^{(f_i+g_j-C_ij)/eps}) (objective.cpp:10-40)."""
    f = _checked(f, problem.n, "dual_value")
    g = _checked(g, problem.m, "dual_value")
    out = ctypes.c_double()
    _check(lib().sknr_dual_value(problem.handle, _ptr(f), _ptr(g), ctypes.byref(out)))
    return out.value


def semi_dual_hessian_quadform(problem: Problem, f, u) -> float:
    """u^T H(f) u of the semi-dual (objective.cpp:53-77)."""
    f = _checked(f, problem.n, "ctransform_of_f")
    u = _vec(u)
    if u.size != problem.n:
        raise ValueError("semi_dual_hessian_quadform: length mismatch")
    out = ctypes.c_double()
    _check(lib().sknr_semi_dual_hessian_quadform(problem.handle, _ptr(f), _ptr(u), ctypes.byref(out)))
    return out.value


def semi_dual_gradient(problem: Problem, f) -> np.ndarray:
    """alpha - row marginal at (f, f^{C,eps}) (objective.cpp:47-51)."""
    g = ctransform_of_f(problem, f)
    row, _, _, _ = plan_marginals(problem, f, g)
    return problem._alpha - row


def restricted_derivatives(problem: Problem, f, basis: SpectralBasis, g=None):
    """(grad, hess) of t -> Q(f + V t) at 0 (objective.cpp:110-148)."""
    if basis.dim != problem.n:
        raise ValueError("restricted_derivatives: basis dimension mismatch")
    if basis.ell < 1:
        raise ValueError("restricted_derivatives: empty basis")
    f = _checked(f, problem.n, "restricted_derivatives(f)")
    if g is None:
        g = ctransform_of_f(problem, f)
    g = _checked(g, problem.m, "restricted_derivatives(g)")
    V = _mat_f(basis.vectors)
    ell = V.shape[1]
    grad = np.empty(ell)
    hess = np.empty((ell, ell), order="F")
    _check(lib().sknr_restricted_derivatives(problem.handle, _ptr(f), _ptr(g), _ptr(V), ell,
                                             _ptr(grad), _ptr(hess)))
    return grad, hess


# ---------------------------------------------------------------- spectral.hpp
def apply_R(problem: Problem, f, g, g1) -> np.ndarray:
    """(R g1)_i = sum_j e^{(f_i+g_j-C_ij)/eps} b_j g1_j (spectral.cpp:29-43)."""
    f = _checked(f, problem.n, "SinkhornOperator(f)")
    g = _checked(g, problem.m, "SinkhornOperator(g)")
    g1 = _vec(g1)
    if g1.size != problem.m:
        raise ValueError("apply_R: length mismatch")
    out = np.empty(problem.n)
    _check(lib().sknr_apply_R(problem.handle, _ptr(f), _ptr(g), _ptr(g1), _ptr(out)))
    return out


def apply_Rt(problem: Problem, f, g, f1) -> np.ndarray:
    """(R^T f1)_j = sum_i e^{(f_i+g_j-C_ij)/eps} a_i f1_i (spectral.cpp:45-62)."""
    f = _checked(f, problem.n, "SinkhornOperator(f)")
    g = _checked(g, problem.m, "SinkhornOperator(g)")
    f1 = _vec(f1)
    if f1.size != problem.n:
        raise ValueError("apply_Rt: length mismatch")
    out = np.empty(problem.m)
    _check(lib().sknr_apply_Rt(problem.handle, _ptr(f), _ptr(g), _ptr(f1), _ptr(out)))
    return out


def apply_K(problem: Problem, f, g, f1, g1):
    """(apply_R(g1), apply_Rt(f1)) (spectral.cpp:64-66)."""
    return apply_R(problem, f, g, g1), apply_Rt(problem, f, g, f1)


def apply_sym_block(problem: Problem, f, g, v) -> np.ndarray:
    f, g, v = _vec(f), _vec(g), _mat_f(v)
    out = np.empty((problem.n, v.shape[1]), order="F")
    _check(lib().sknr_apply_sym_block(problem.handle, _ptr(f), _ptr(g), _ptr(v), v.shape[1], _ptr(out)))
    return out


def apply_sym_t_block(problem: Problem, f, g, u) -> np.ndarray:
    f, g, u = _vec(f), _vec(g), _mat_f(u)
    out = np.empty((problem.m, u.shape[1]), order="F")
    _check(lib().sknr_apply_sym_t_block(problem.handle, _ptr(f), _ptr(g), _ptr(u), u.shape[1],
                                        _ptr(out)))
    return out


def top_modes(problem: Problem, f, g, ell: int, tol: float = 1e-8,
              max_power_iters: int = -1, method: str = "subspace", degree: int = 8) -> SpectralBasis:
    """top_modes (spectral.cpp:125-193). method="subspace" is the reference's block
    subspace iteration; method="chebyshev" (opt-in, not in the reference) filters
    each step with a degree-`degree` Chebyshev polynomial -- same Rayleigh-Ritz,
    same residual criterion, far fewer operator applications on clustered spectra;
    method="lanczos" (opt-in) runs restarted block Lanczos with `degree` blocks per
    cycle and the same explicit residual test."""
    f = _checked(f, problem.n, "SinkhornOperator(f)")
    g = _checked(g, problem.m, "SinkhornOperator(g)")
    ell = int(ell)
    if ell < 1:
        raise ValueError("top_modes: ell must be >= 1")
    if ell >= problem.n:
        raise ValueError("top_modes: ell must be < n")
    vec = np.empty((problem.n, ell), order="F")
    vsym = np.empty((problem.n, ell), order="F")
    rhos = np.empty(ell)
    sweeps = _I64()
    methods = {"subspace": 0, "chebyshev": 1, "lanczos": 2}
    if method not in methods:
        raise ValueError("top_modes: method must be subspace|chebyshev|lanczos")
    _check(lib().sknr_top_modes_ex(problem.handle, _ptr(f), _ptr(g), ell, float(tol), int(max_power_iters),
                                   methods[method], int(degree), _ptr(vec), _ptr(vsym), _ptr(rhos),
                                   ctypes.byref(sweeps)))
    return SpectralBasis(vec, vsym, rhos, problem.epsilon, int(sweeps.value))


def spectrum(problem: Problem, f, g, k: int, vectors: bool = False, tol: float = 1e-8,
             max_power_iters: int = -1) -> dict:
    """spectrum_report (spectral.cpp:195-228) as the reference binding's dict
    (bindings.cpp:118-136): epsilon, rho, eigenvalues_of_K (+rho, -rho),
    hessian_eigs_low/high = (1 -+ rho)/eps and, with vectors, vectors_f (n x k)
    and vectors_g (m x k)."""
    f = _checked(f, problem.n, "SinkhornOperator(f)")
    g = _checked(g, problem.m, "SinkhornOperator(g)")
    k = int(k)
    if k < 1 or k > min(problem.n, problem.m) - 1:
        raise ValueError("spectrum_report: need 1 <= k <= min(n,m)-1")
    rho, lo, hi = np.empty(k), np.empty(k), np.empty(k)
    vf = np.empty((problem.n, k), order="F") if vectors else None
    vg = np.empty((problem.m, k), order="F") if vectors else None
    _check(lib().sknr_spectrum_report(problem.handle, _ptr(f), _ptr(g), k, 1 if vectors else 0, float(tol),
                                      int(max_power_iters), _ptr(rho), _ptr(lo), _ptr(hi), _ptr(vf), _ptr(vg)))
    out = {"epsilon": problem.epsilon, "rho": rho, "eigenvalues_of_K": [(float(r), float(-r)) for r in rho],
           "hessian_eigs_low": lo, "hessian_eigs_high": hi}
    if vectors:
        out["vectors_f"] = vf
        out["vectors_g"] = vg
    return out


def projector_distance(basis_a: SpectralBasis, basis_b: SpectralBasis) -> float:
    """||P_A - P_B||_2 = ||(I - A A^T) B||_2 in symmetrised coordinates (spectral.cpp:230-242)."""
    a, b = _mat_f(basis_a.vectors_sym), _mat_f(basis_b.vectors_sym)
    if a.shape != b.shape:
        raise ValueError("projector_distance: dimension mismatch")
    out = ctypes.c_double()
    _check(lib().sknr_projector_distance(a.shape[0], a.shape[1], _ptr(a), _ptr(b), ctypes.byref(out)))
    return out.value


# ---------------------------------------------------------------- solver.hpp
@dataclass
class NewtonOutcome:
    """NewtonOutcome (solver.hpp:50-57)."""

    f: np.ndarray
    accepted: bool
    factorization_failed: bool


def sk_sweep(problem: Problem, f, g=None):
    """One Sinkhorn sweep, g-then-f (solver.cpp:12-17): returns (f', g')."""
    g1 = ctransform_of_f(problem, f)
    return ctransform_of_g(problem, g1), g1


def newton_step(problem: Problem, f, basis: SpectralBasis, accept: str = "literal") -> NewtonOutcome:
    """One restricted Newton step from f (solver.cpp:59-69); `accept` as in solve()."""
    if basis.ell < 1:
        raise ValueError("newton_step: empty basis")
    f = _checked(f, problem.n, "ctransform_of_f")
    V = _mat_f(basis.vectors)
    if V.shape[0] != problem.n:
        raise ValueError("restricted_derivatives: basis dimension mismatch")
    fo = np.empty(problem.n)
    acc, fail = ctypes.c_int(), ctypes.c_int()
    _check(lib().sknr_newton_step_ex(problem.handle, _ptr(f), _ptr(V), V.shape[1], _accept_code(accept),
                                     _ptr(fo), ctypes.byref(acc), ctypes.byref(fail)))
    return NewtonOutcome(fo, bool(acc.value), bool(fail.value))


_ACCEPT = {"literal": 0, "stable": 1}


def _accept_code(accept) -> int:
    if accept not in _ACCEPT:
        raise ValueError("accept must be 'literal' or 'stable'")
    return _ACCEPT[accept]


# records preallocated per solve; longer traces are fetched whole afterwards (sknr_last_trace)
_TRACE_PREALLOC = 4096


def _full_trace(problem, recs, cap, total):
    if total <= cap:
        return _records(recs, total)
    buf = (_Record * total)()
    got = _I64()
    _check(lib().sknr_last_trace(problem.handle, buf, total, ctypes.byref(got)))
    return _records(buf, min(total, got.value))


def _config(tol, max_iter, ell, trace, newton=True, exact_marginals=False, accept="literal") -> _Config:
    c = _Config()
    lib().sknr_config_default(ctypes.byref(c))
    c.tol_omega = float(tol)
    c.max_iter = int(max_iter)
    c.ell = int(ell)
    c.trace_enabled = 1 if trace else 0
    c.newton_enabled = 1 if newton else 0
    c.exact_marginals = 1 if exact_marginals else 0
    c.accept_test = _accept_code(accept)
    return c


def solve(problem: Problem, tol: float = 1e-9, max_iter: int = 100000, ell: int = 0,
          basis: Optional[SpectralBasis] = None, init=None, trace: bool = True,
          exact_marginals: bool = False, accept: str = "literal") -> SolveResult:
    """SK-NR(ell) (Alg. 1; solver.cpp:71-156). exact_marginals=True evaluates the
    stopping test from explicit plan row/column sums (core.cpp:120-143) instead
    of the fused transform (2 extra passes per iteration).

    accept: the Newton accept test (solver.cpp:46-47). "literal" (the reference)
    compares Q(f') > Q(f) evaluated in full; once the gain of a step falls below
    ulp(Q) that comparison is rounding noise on any platform. "stable" evaluates the
    same predicate as dQ = a.(f'-f) + b.(h'-h) > 0 with h'-h = -eps log1p(...) from an
    anchor pass, whose rounding scales with the step (sknr_config.accept_test)."""
    cfg = _config(tol, max_iter, ell, trace, exact_marginals=exact_marginals, accept=accept)
    V = None
    bell = 0
    if ell > 0:
        if basis is None:
            raise ValueError("solve: ell > 0 requires a basis")
        if basis.ell != ell:
            raise ValueError("solve: basis has wrong column count")
        if basis.dim != problem.n:
            raise ValueError("solve: basis dimension mismatch")
        V = _mat_f(basis.vectors)
        bell = ell
    f0 = g0 = None
    if init is not None:
        f0, g0 = _vec(init[0]), _vec(init[1])
        if f0.size != problem.n or g0.size != problem.m:
            raise ValueError("solve: init potential sizes mismatch")
    f = np.empty(problem.n)
    g = np.empty(problem.m)
    iters = _I64()
    conv = ctypes.c_int()
    cap = min(int(max_iter), _TRACE_PREALLOC) if trace else 0
    recs = (_Record * max(cap, 1))()
    tlen = _I64()
    _check(lib().sknr_solve(problem.handle, ctypes.byref(cfg), _ptr(V), bell, _ptr(f0), _ptr(g0),
                            _ptr(f), _ptr(g), ctypes.byref(iters), ctypes.byref(conv), recs, cap,
                            ctypes.byref(tlen)))
    tr = _full_trace(problem, recs, cap, int(tlen.value)) if trace else []
    return SolveResult(f, g, bool(conv.value), int(iters.value), tr, problem, problem.epsilon)


def solve_batch(problems: Sequence[Problem], tol: float = 1e-9, max_iter: int = 100000, ell: int = 0,
                bases: Optional[Sequence[SpectralBasis]] = None, inits=None,
                exact_marginals: bool = False, accept: str = "literal") -> list:
    """Solve independent problems together (one CUDA graph per iteration, one
    concurrent branch per problem; not in the reference API). Each result equals
    solve(problems[b], ...) bit for bit; traces are not recorded."""
    B = len(problems)
    if B < 1:
        raise ValueError("solve_batch: empty batch")
    cfg = _config(tol, max_iter, ell, False, exact_marginals=exact_marginals, accept=accept)
    handles = (_P * B)(*[p.handle for p in problems])
    keep = []

    def arr(vals):
        out = (_D * B)()
        for b, v in enumerate(vals):
            out[b] = _ptr(v)
        return out

    bptr = None
    if ell > 0:
        if bases is None or len(bases) != B:
            raise ValueError("solve: ell > 0 requires a basis")
        Vs = []
        for p, bs in zip(problems, bases):
            V = _mat_f(bs.vectors)
            if V.shape[0] != p.n:
                raise ValueError("solve: basis dimension mismatch")
            if V.shape[1] != ell:
                raise ValueError("solve: basis has wrong column count")
            Vs.append(V)
        keep.append(Vs)
        bptr = arr(Vs)
    fptr = gptr = None
    if inits is not None:
        fs, gs = [], []
        for p, (f0, g0) in zip(problems, inits):
            f0, g0 = _vec(f0), _vec(g0)
            if f0.size != p.n or g0.size != p.m:
                raise ValueError("solve: init potential sizes mismatch")
            fs.append(f0)
            gs.append(g0)
        keep.append((fs, gs))
        fptr, gptr = arr(fs), arr(gs)
    fo = [np.empty(p.n) for p in problems]
    go = [np.empty(p.m) for p in problems]
    iters = (_I64 * B)()
    conv = (ctypes.c_int * B)()
    _check(lib().sknr_solve_batch(handles, B, ctypes.byref(cfg), bptr, int(ell), fptr, gptr, arr(fo), arr(go),
                                  iters, conv))
    return [SolveResult(fo[b], go[b], bool(conv[b]), int(iters[b]), [], problems[b], problems[b].epsilon)
            for b in range(B)]


def solve_small_batch(problems, tol: float = 1e-9, max_iter: int = 100000) -> list:
    """Plain SK (ell = 0, from f = 0) for small point-cloud problems in ONE kernel launch
    (one dimension d <= 4; n, m <= 8192 at d <= 2, 6224 at d = 3, 4979 at d = 4): one
    CTA per problem when the batch fills the GPU, a cooperative group of CTAs per
    problem otherwise (a single problem is the low-latency solve). `problems` holds
    PointProblem objects or (x, y, alpha, beta, epsilon[, cost_scale]) tuples. Same
    iteration and stopping test as solve(); reductions run in a different order, so
    potentials agree with solve() to rounding, not bit for bit. Not in the reference."""
    items = []
    for p in problems:
        if isinstance(p, PointProblem):
            items.append((p._x, p._y, p._alpha, p._beta, p.epsilon, p._cost_scale))
        else:
            x, y, a, b, e = p[:5]
            items.append((_mat_f(x), _mat_f(y), _vec(a), _vec(b), float(e), float(p[5]) if len(p) > 5 else 1.0))
    B = len(items)
    if B < 1:
        raise ValueError("solve_small_batch: empty batch")
    d = items[0][0].shape[1] if items[0][0].ndim == 2 else 1
    keep = []

    def col(a):
        a = _mat_f(a)
        if a.ndim == 1:
            a = a.reshape(-1, 1, order="F")
        keep.append(a)
        return a

    xs = [col(it[0]) for it in items]
    ys = [col(it[1]) for it in items]
    for x_, y_ in zip(xs, ys):
        if x_.shape[1] != d or y_.shape[1] != d:
            raise ValueError("solve_small_batch: all problems need the same dimension")
    n = (_I64 * B)(*[x_.shape[0] for x_ in xs])
    m = (_I64 * B)(*[y_.shape[0] for y_ in ys])
    av = [_vec(it[2]) for it in items]
    bv = [_vec(it[3]) for it in items]
    eps = np.array([it[4] for it in items], dtype=np.float64)
    cs = np.array([it[5] for it in items], dtype=np.float64)
    fo = [np.empty(x_.shape[0]) for x_ in xs]
    go = [np.empty(y_.shape[0]) for y_ in ys]

    def arr(vals):
        out = (_D * B)()
        for k, v in enumerate(vals):
            out[k] = _ptr(v)
        return out

    iters = (_I64 * B)()
    conv = (ctypes.c_int * B)()
    _check(lib().sknr_solve_small_batch(B, d, n, m, arr(xs), arr(ys), arr(av), arr(bv), _ptr(eps), _ptr(cs),
                                        float(tol), int(max_iter), arr(fo), arr(go), iters, conv))
    return [SolveResult(fo[k], go[k], bool(conv[k]), int(iters[k]), []) for k in range(B)]


def anneal(problem: Problem, epsilons: Sequence[float], warm: str = "spectral", ell: int = 8,
           refresh_basis: bool = False, tol: float = 1e-9, max_iter: int = 100000,
           accept: str = "literal") -> list:
    """Epsilon-annealing driver (solver.cpp:158-222); `accept` as in solve()."""
    modes = {"none": 0, "potentials": 1, "spectral": 2}
    if warm not in modes:
        raise ValueError("warm must be none|potentials|spectral")
    eps = _vec(epsilons)
    S = eps.size
    if S == 0:
        raise ValueError("anneal: empty schedule")
    cfg = _config(tol, max_iter, ell, True, accept=accept)
    n, m = problem.n, problem.m
    F = np.empty(S * n)
    G = np.empty(S * m)
    iters = (_I64 * S)()
    conv = (ctypes.c_int * S)()
    cap = min(int(max_iter), _TRACE_PREALLOC) * S
    recs = (_Record * max(cap, 1))()
    offs = (_I64 * S)()
    tlen = _I64()
    _check(lib().sknr_anneal(problem.handle, _ptr(eps), S, modes[warm], 1 if refresh_basis else 0,
                             ctypes.byref(cfg), _ptr(F), _ptr(G), iters, conv, recs, cap, offs,
                             ctypes.byref(tlen)))
    if tlen.value > cap:
        cap = int(tlen.value)
        recs = (_Record * cap)()
        got = _I64()
        _check(lib().sknr_last_trace(problem.handle, recs, cap, ctypes.byref(got)))
    out = []
    for s in range(S):
        lo = offs[s]
        hi = offs[s + 1] if s + 1 < S else tlen.value
        out.append(SolveResult(F[s * n:(s + 1) * n].copy(), G[s * m:(s + 1) * m].copy(), bool(conv[s]),
                               int(iters[s]), _records(recs[lo:min(hi, cap)], hi - lo), problem,
                               float(eps[s])))
    return out


# ---------------------------------------------------------------- measurement
def set_tensor_block_pass(on: bool) -> bool:
    """Select the tensor-core (tcgen05 int8 slice) Newton block pass (default) or the FP64
    DMMA pass for plans made afterwards; returns the previous setting."""
    prev = bool(lib().sknr_get_tensor_block_pass())
    _check(lib().sknr_set_tensor_block_pass(1 if on else 0))
    return prev


def probe_i8_mma(A: np.ndarray, Bt: np.ndarray) -> np.ndarray:
    """D = A @ Bt.T on one tcgen05 int8 GEMM (A: 128 x k uint8, Bt: n x k int8)."""
    A = np.ascontiguousarray(A, dtype=np.uint8)
    Bt = np.ascontiguousarray(Bt, dtype=np.int8)
    n, k = Bt.shape
    if A.shape != (128, k):
        raise ValueError("probe_i8_mma: A must be 128 x k")
    D = np.zeros((128, n), dtype=np.int32)
    rc = lib().sknr_probe_i8_mma(A.ctypes.data, Bt.ctypes.data, n, k, D.ctypes.data)
    if rc != 0:
        raise RuntimeError(f"probe_i8_mma failed ({rc})")
    return D


def bench_pass(problem: Problem, which: int, ell: int = 0, passes: int = 5):
    ms, kms = ctypes.c_double(), ctypes.c_double()
    _check(lib().sknr_bench_pass(problem.handle, int(which), int(ell), int(passes), ctypes.byref(ms),
                                 ctypes.byref(kms)))
    return ms.value, kms.value


def bench_iterations(problem: Problem, ell: int = 0, basis: Optional[SpectralBasis] = None,
                     iters: int = 5, warmup: int = 1, flush_l2: bool = True, accept: str = "literal"):
    """Device ms per SK-NR(ell) iteration (CUDA events per iteration, L2 flushed
    between iterations) and the number of kernels in one iteration."""
    cfg = _config(1e-9, 1 << 40, ell, False, accept=accept)
    V = _mat_f(basis.vectors) if (basis is not None and ell > 0) else None
    ms = ctypes.c_double()
    kpi = _I64()
    _check(lib().sknr_bench_iterations(problem.handle, ctypes.byref(cfg), _ptr(V),
                                       int(ell) if V is not None else 0, int(warmup), int(iters),
                                       1 if flush_l2 else 0, ctypes.byref(ms), ctypes.byref(kpi)))
    return ms.value, int(kpi.value)


# ---------------------------------------------------------------- row sharding (multi-GPU)
def comm_unique_id() -> bytes:
    """NCCL unique id (rank 0), to be shared with the other ranks out of band."""
    buf = (ctypes.c_ubyte * 128)()
    _check(lib().sknr_comm_unique_id(buf))
    return bytes(buf)


def comm_init(rank: int, world: int, uid: bytes, device: int = -1) -> None:
    """One process per GPU: join the NCCL communicator used by sharded problems."""
    if len(uid) != 128:
        raise ValueError("comm_init: unique id must be 128 bytes")
    buf = (ctypes.c_ubyte * 128).from_buffer_copy(uid)
    _check(lib().sknr_comm_init(int(rank), int(world), buf, int(device)))


def comm_stats(reset: bool = False):
    """(calls, bytes) of the collectives this process issued for sharded handles."""
    c, b = _I64(), _I64()
    _check(lib().sknr_comm_stats(ctypes.byref(c), ctypes.byref(b), 1 if reset else 0))
    return int(c.value), int(b.value)


def comm_destroy() -> None:
    _check(lib().sknr_comm_destroy())


def comm_init_emulated(world: int) -> None:
    """Testing aid: `world` in-process emulated ranks on this GPU. Shard R handles
    (one per rank) after this call and drive each from its own thread; collectives
    are exchanged in-process (see sknr_comm_init_emulated)."""
    _check(lib().sknr_comm_init_emulated(int(world)))


def run_emulated_shards(make_problem, world: int, fn):
    """Run fn(problem_r) for r = 0..world-1 on emulated shards, one thread per rank;
    returns the per-rank results. make_problem() builds a fresh full problem."""
    import threading

    comm_init_emulated(world)
    try:
        probs = []
        for r in range(world):
            p = make_problem()
            shard(p, r, world)
            probs.append(p)
        out = [None] * world
        err = [None] * world

        def run(r):
            try:
                out[r] = fn(probs[r])
            except BaseException as e:  # noqa: BLE001 -- re-raised in the caller
                err[r] = e

        threads = [threading.Thread(target=run, args=(r,)) for r in range(world)]
        for th in threads:
            th.start()
        for th in threads:
            th.join()
        for e in err:
            if e is not None:
                raise e
        return out
    finally:
        comm_destroy()


def row_partition(n: int, world: int, rank: int):
    """Rows [n*r/R, n*(r+1)/R) of rank r (the partition sknr_problem_shard enforces)."""
    return n * rank // world, n * (rank + 1) // world


def shard(problem: Problem, rank: int, world: int) -> None:
    """Keep only this rank's source rows on the device (C ABI sknr_problem_shard).
    Inputs and outputs of every call stay full length on every rank."""
    b, e = row_partition(problem.n, world, rank)
    _check(lib().sknr_problem_shard(problem.handle, b, e))
    problem._rows = (b, e)


def debug_counters(problem: Problem) -> dict:
    out = (_I64 * 6)()
    _check(lib().sknr_debug_counters(problem.handle, out))
    return {"exact_col": out[0], "exact_row": out[1], "retry_col": out[2], "retry_row": out[3],
            "cull_tested": out[4], "cull_kept": out[5]}


def tune_variant(problem: Problem, variant: int, passes: int = 5) -> float:
    ms = ctypes.c_double()
    _check(lib().sknr_tune_variant(problem.handle, int(variant), int(passes), ctypes.byref(ms)))
    return ms.value


def bench_fp64_peak():
    """(TFLOP/s, ms) of a DFMA-only kernel filling every SM: the measured FP64 ceiling."""
    t, ms = ctypes.c_double(), ctypes.c_double()
    _check(lib().sknr_bench_fp64_peak(ctypes.byref(t), ctypes.byref(ms)))
    return t.value, ms.value


def bench_mufu_peak():
    """(G ex2/s, ms) of an ex2.approx.f32-only kernel filling every SM: the MUFU ceiling
    of the fp32 sum pass (set_precision(32))."""
    t, ms = ctypes.c_double(), ctypes.c_double()
    _check(lib().sknr_bench_mufu_peak(ctypes.byref(t), ctypes.byref(ms)))
    return t.value, ms.value


# ---------------------------------------------------------------- harness (bindings.cpp:180-215)
def oracle_solve(problem: Problem, target_residual: float = 1e-13):
    """Ground-truth desk-scale solve (oracle.cpp:21-90); see harness.oracle_solve."""
    from .harness import oracle_solve as _os
    return _os(problem, target_residual)


def gaussian_cloud(count: int, mean, cov, seed: int):
    """(points n x 2, uniform weights) drawn as generators.cpp:19-36."""
    from .generators import gaussian_cloud as _gc
    return _gc(count, mean, cov, seed)


def sq_euclidean_cost(source, target) -> np.ndarray:
    """Dense ||x_i - y_j||^2 (generators.cpp:94-103); the solver itself never stores it
    for point clouds (PointProblem)."""
    from .generators import sq_euclidean_cost as _sq
    return _sq(np.asarray(source, dtype=np.float64), np.asarray(target, dtype=np.float64))


__all__ = [
    "EigensolverError", "IterationRecord", "NewtonOutcome", "PointProblem", "Problem", "SolveResult",
    "SpectralBasis", "__version__", "anneal", "apply_K", "apply_R", "apply_Rt", "apply_sym_block",
    "apply_sym_t_block", "coupling", "coupling_rows", "ctransform_of_f", "dual_value", "gauge_distance",
    "gauge_normalized", "marginal_gap", "newton_step", "projector_distance", "semi_dual_hessian_quadform",
    "sk_sweep", "solve_batch", "solve_small_batch", "spectrum", "oracle_solve", "gaussian_cloud", "sq_euclidean_cost",
    "ctransform_of_g", "kernel_launch_count", "lib", "log_sum_exp", "marginal_error", "osc_norm",
    "plan_marginals", "restricted_derivatives", "comm_init", "comm_unique_id", "comm_destroy",
    "row_partition", "shard", "comm_init_emulated", "run_emulated_shards", "semi_dual_gradient", "semi_dual_value", "solve",
    "top_modes", "version",
]
