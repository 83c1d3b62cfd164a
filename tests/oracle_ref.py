"""ctypes binding of the CPU oracle (oracle/liboracle.so) -- TEST INFRASTRUCTURE ONLY.

The oracle is a plain C++ restatement of the reference SK-NR path
(oracle/sknr_oracle.cpp cites reference file:line per function). Tests use it
as the checker for the GPU library; nothing in the product package imports it.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "oracle", "liboracle.so")
_D = ctypes.POINTER(ctypes.c_double)
_lib = None


class OracleProblem(ctypes.Structure):
    _fields_ = [
        ("kind", ctypes.c_int),
        ("cost", _D),
        ("x", _D),
        ("y", _D),
        ("n", ctypes.c_long),
        ("m", ctypes.c_long),
        ("d", ctypes.c_long),
        ("cost_div", ctypes.c_double),
        ("alpha", _D),
        ("beta", _D),
        ("eps", ctypes.c_double),
    ]


class OracleRecord(ctypes.Structure):
    _fields_ = [
        ("marginal_error", ctypes.c_double),
        ("marginal_error_inf", ctypes.c_double),
        ("semi_dual_value", ctypes.c_double),
        ("newton_attempted", ctypes.c_int),
        ("newton_accepted", ctypes.c_int),
        ("newton_gain", ctypes.c_double),
        ("newton_step_max", ctypes.c_double),
    ]


def build():
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build()
        _lib = ctypes.CDLL(LIB)
        _lib.oracle_last_error.restype = ctypes.c_char_p
        # output-parallel loops are bitwise identical to 1 thread (sknr_oracle.cpp header)
        _lib.oracle_set_threads(int(os.environ.get("ORACLE_THREADS", "0")))
    return _lib


def set_threads(t: int):
    lib().oracle_set_threads(int(t))


def set_accept_mode(mode) -> None:
    """Accept test of try_newton: "literal" (the reference's Q(f') > Q(f)) or "stable"
    (the same predicate evaluated as dQ > 0, sknr_oracle.cpp stable_delta_q)."""
    lib().oracle_set_accept_mode(1 if mode in ("stable", 1) else 0)


class accept_mode:
    """Context manager: run oracle calls under one accept mode, restore literal after."""

    def __init__(self, mode):
        self.mode = mode

    def __enter__(self):
        set_accept_mode(self.mode)
        return self

    def __exit__(self, *exc):
        set_accept_mode("literal")
        return False


def max_threads() -> int:
    return int(lib().oracle_max_threads())


def _p(a):
    return None if a is None else a.ctypes.data_as(_D)


class Instance:
    """Keeps numpy buffers alive for an OracleProblem."""

    def __init__(self, alpha, beta, eps, cost=None, x=None, y=None, cost_div=1.0):
        self.alpha = np.ascontiguousarray(alpha, dtype=np.float64)
        self.beta = np.ascontiguousarray(beta, dtype=np.float64)
        self.eps = float(eps)
        self.cost = None if cost is None else np.asfortranarray(cost, dtype=np.float64)
        self.x = None if x is None else np.asfortranarray(x, dtype=np.float64)
        self.y = None if y is None else np.asfortranarray(y, dtype=np.float64)
        n = self.alpha.size
        m = self.beta.size
        self.n, self.m = n, m
        self.s = OracleProblem()
        self.s.kind = 0 if cost is not None else 1
        self.s.cost = _p(self.cost)
        self.s.x = _p(self.x)
        self.s.y = _p(self.y)
        self.s.n = n
        self.s.m = m
        self.s.d = 0 if self.x is None else self.x.shape[1]
        self.s.cost_div = float(cost_div)
        self.s.alpha = _p(self.alpha)
        self.s.beta = _p(self.beta)
        self.s.eps = self.eps

    def with_epsilon(self, eps):
        return Instance(self.alpha, self.beta, eps, self.cost, self.x, self.y, self.s.cost_div)


def _check(rc):
    if rc == 0:
        return
    msg = lib().oracle_last_error().decode()
    if rc == 1:
        raise ValueError(msg)
    if rc == 2:
        raise RuntimeError("EigensolverError: " + msg)
    raise RuntimeError(msg)


def log_sum_exp(values, lw):
    v = np.ascontiguousarray(values, dtype=np.float64)
    w = np.ascontiguousarray(lw, dtype=np.float64)
    out = ctypes.c_double()
    _check(lib().oracle_log_sum_exp(_p(v), _p(w), ctypes.c_long(v.size), ctypes.byref(out)))
    return out.value


def ctransform_of_f(P: Instance, f):
    f = np.ascontiguousarray(f, dtype=np.float64)
    g = np.empty(P.m)
    _check(lib().oracle_ctransform_f(ctypes.byref(P.s), _p(f), _p(g)))
    return g


def ctransform_of_g(P: Instance, g):
    g = np.ascontiguousarray(g, dtype=np.float64)
    f = np.empty(P.n)
    _check(lib().oracle_ctransform_g(ctypes.byref(P.s), _p(g), _p(f)))
    return f


def plan_marginals(P: Instance, f, g):
    f = np.ascontiguousarray(f, dtype=np.float64)
    g = np.ascontiguousarray(g, dtype=np.float64)
    row, col = np.empty(P.n), np.empty(P.m)
    l2, inf = ctypes.c_double(), ctypes.c_double()
    _check(lib().oracle_plan_marginals(ctypes.byref(P.s), _p(f), _p(g), _p(row), _p(col),
                                       ctypes.byref(l2), ctypes.byref(inf)))
    return row, col, l2.value, inf.value


def coupling(P: Instance, f, g):
    f = np.ascontiguousarray(f, dtype=np.float64)
    g = np.ascontiguousarray(g, dtype=np.float64)
    plan = np.empty((P.n, P.m), order="F")
    _check(lib().oracle_coupling(ctypes.byref(P.s), _p(f), _p(g), _p(plan)))
    return plan


def semi_dual_value(P: Instance, f):
    f = np.ascontiguousarray(f, dtype=np.float64)
    out = ctypes.c_double()
    _check(lib().oracle_semi_dual_value(ctypes.byref(P.s), _p(f), ctypes.byref(out)))
    return out.value


def restricted_derivatives(P: Instance, f, g, V):
    f = np.ascontiguousarray(f, dtype=np.float64)
    g = np.ascontiguousarray(g, dtype=np.float64)
    V = np.asfortranarray(V, dtype=np.float64)
    ell = V.shape[1]
    grad = np.empty(ell)
    hess = np.empty((ell, ell), order="F")
    _check(lib().oracle_restricted_derivatives(ctypes.byref(P.s), _p(f), _p(g), _p(V),
                                               ctypes.c_long(ell), _p(grad), _p(hess)))
    return grad, hess


def apply_sym_block(P: Instance, f, g, V):
    f = np.ascontiguousarray(f, dtype=np.float64)
    g = np.ascontiguousarray(g, dtype=np.float64)
    V = np.asfortranarray(V, dtype=np.float64)
    out = np.empty((P.n, V.shape[1]), order="F")
    _check(lib().oracle_apply_sym_block(ctypes.byref(P.s), _p(f), _p(g), _p(V),
                                        ctypes.c_long(V.shape[1]), _p(out)))
    return out


def apply_sym_t_block(P: Instance, f, g, U):
    f = np.ascontiguousarray(f, dtype=np.float64)
    g = np.ascontiguousarray(g, dtype=np.float64)
    U = np.asfortranarray(U, dtype=np.float64)
    out = np.empty((P.m, U.shape[1]), order="F")
    _check(lib().oracle_apply_sym_t_block(ctypes.byref(P.s), _p(f), _p(g), _p(U),
                                          ctypes.c_long(U.shape[1]), _p(out)))
    return out


def apply_R(P: Instance, f, g, g1):
    f, g, g1 = (np.ascontiguousarray(v, dtype=np.float64) for v in (f, g, g1))
    out = np.empty(P.n)
    _check(lib().oracle_apply_R(ctypes.byref(P.s), _p(f), _p(g), _p(g1), _p(out)))
    return out


def apply_Rt(P: Instance, f, g, f1):
    f, g, f1 = (np.ascontiguousarray(v, dtype=np.float64) for v in (f, g, f1))
    out = np.empty(P.m)
    _check(lib().oracle_apply_Rt(ctypes.byref(P.s), _p(f), _p(g), _p(f1), _p(out)))
    return out


def dual_value(P: Instance, f, g):
    f, g = (np.ascontiguousarray(v, dtype=np.float64) for v in (f, g))
    out = ctypes.c_double()
    _check(lib().oracle_dual_value(ctypes.byref(P.s), _p(f), _p(g), ctypes.byref(out)))
    return out.value


def semi_dual_hessian_quadform(P: Instance, f, u):
    f, u = (np.ascontiguousarray(v, dtype=np.float64) for v in (f, u))
    out = ctypes.c_double()
    _check(lib().oracle_semi_dual_hessian_quadform(ctypes.byref(P.s), _p(f), _p(u), ctypes.byref(out)))
    return out.value


def newton_step(P: Instance, f, V):
    f = np.ascontiguousarray(f, dtype=np.float64)
    V = np.asfortranarray(V, dtype=np.float64)
    fo = np.empty(P.n)
    acc, fail = ctypes.c_int(), ctypes.c_int()
    _check(lib().oracle_newton_step(ctypes.byref(P.s), _p(f), _p(V), ctypes.c_long(V.shape[1]), _p(fo),
                                    ctypes.byref(acc), ctypes.byref(fail)))
    return fo, bool(acc.value), bool(fail.value)


def top_modes(P: Instance, f, g, ell, tol=1e-8, max_power_iters=-1):
    f = np.ascontiguousarray(f, dtype=np.float64)
    g = np.ascontiguousarray(g, dtype=np.float64)
    vec = np.empty((P.n, ell), order="F")
    vsym = np.empty((P.n, ell), order="F")
    rhos = np.empty(ell)
    best = ctypes.c_double()
    sweeps = ctypes.c_long()
    _check(lib().oracle_top_modes(ctypes.byref(P.s), _p(f), _p(g), ctypes.c_long(ell),
                                  ctypes.c_double(tol), ctypes.c_long(max_power_iters), _p(vec),
                                  _p(vsym), _p(rhos), ctypes.byref(best), ctypes.byref(sweeps)))
    return {"vectors": vec, "vectors_sym": vsym, "rhos": rhos, "sweeps": sweeps.value,
            "best_residual": best.value}


def solve(P: Instance, tol=1e-9, max_iter=100000, ell=0, V=None, init=None, trace=True,
          trace_cap=None):
    f = np.empty(P.n)
    g = np.empty(P.m)
    iters = ctypes.c_long()
    conv = ctypes.c_int()
    cap = int(trace_cap if trace_cap is not None else max_iter)
    recs = (OracleRecord * max(cap, 1))()
    tlen = ctypes.c_long()
    Vp = None if V is None else np.asfortranarray(V, dtype=np.float64)
    f0 = g0 = None
    if init is not None:
        f0 = np.ascontiguousarray(init[0], dtype=np.float64)
        g0 = np.ascontiguousarray(init[1], dtype=np.float64)
    _check(lib().oracle_solve(ctypes.byref(P.s), ctypes.c_double(tol), ctypes.c_long(max_iter),
                              ctypes.c_long(ell), _p(Vp), _p(f0), _p(g0), ctypes.c_int(1 if trace else 0),
                              _p(f), _p(g), ctypes.byref(iters), ctypes.byref(conv), recs,
                              ctypes.c_long(cap), ctypes.byref(tlen)))
    tr = [(r.marginal_error, r.marginal_error_inf, r.semi_dual_value, r.newton_attempted,
           r.newton_accepted, r.newton_gain, r.newton_step_max) for r in recs[:min(tlen.value, cap)]]
    return {"f": f, "g": g, "iterations": iters.value, "converged": bool(conv.value), "trace": tr}


def anneal(P: Instance, epsilons, warm="spectral", ell=8, refresh_basis=False, tol=1e-9,
           max_iter=100000):
    """anneal (solver.cpp:158-222) composed from the oracle's solve and top_modes."""
    eps = list(epsilons)
    for s in range(1, len(eps)):
        if not eps[s] < eps[s - 1]:
            raise ValueError("anneal: epsilons must be strictly decreasing")
    results = [solve(P.with_epsilon(eps[0]), tol, max_iter)]
    basis = None
    for s in range(1, len(eps)):
        prev = results[-1]
        use_ell = 0
        V = None
        if warm == "spectral" and ell > 0:
            if basis is None or refresh_basis:
                basis = top_modes(P.with_epsilon(eps[s - 1]), prev["f"], prev["g"], ell)
            use_ell = ell
            V = basis["vectors"]
        init = None if warm == "none" else (prev["f"], prev["g"])
        results.append(solve(P.with_epsilon(eps[s]), tol, max_iter, use_ell, V, init))
    return results


def sym_eig(A):
    A = np.asfortranarray(A, dtype=np.float64)
    k = A.shape[0]
    ev = np.empty(k)
    V = np.empty((k, k), order="F")
    _check(lib().oracle_sym_eig(_p(A), ctypes.c_long(k), _p(ev), _p(V)))
    return ev, V
