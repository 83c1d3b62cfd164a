"""Tensor-core Newton block pass (i8_kernels.cu): tcgen05 int8 GEMMs over exact byte slices.

The restricted derivatives (objective.cpp:110-142: S = V^T P~, r = P~ beta, then the l x l
system) are computed once with the tensor-core pass and once with the FP64 DMMA pass, and
both are checked against the oracle at the tolerances of test_gpu_parity.py; the encoding
itself (descriptors, operand layouts, TMEM read-back) is pinned by an exact int8 GEMM.
"""
import numpy as np
import pytest

import oracle_ref as O
import paper_2506_14780_b200 as sk
from paper_2506_14780_b200 import generators as G
from support import rel_err, smooth_basis

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,k", [(32, 32), (224, 64), (256, 256), (96, 128)])
def test_probe_i8_mma_is_exact(n, k):
    rng = np.random.default_rng(n * 1000 + k)
    A = rng.integers(0, 256, (128, k), dtype=np.uint8)
    Bt = rng.integers(-128, 128, (n, k), dtype=np.int8)
    D = sk.probe_i8_mma(A, Bt)
    ref = A.astype(np.int64) @ Bt.astype(np.int64).T
    assert np.array_equal(D.astype(np.int64), ref)


def _points(d, n, m, seed):
    rng = np.random.default_rng(seed)
    x = np.asfortranarray(rng.uniform(0, 1, (n, d)))
    y = np.asfortranarray(rng.uniform(0, 1, (m, d)))
    a = rng.uniform(0.5, 1.5, n)
    a /= a.sum()
    b = rng.uniform(0.5, 1.5, m)
    b /= b.sum()
    return rng, x, y, a, b


def _both_paths(fn):
    prev = sk.set_tensor_block_pass(True)
    try:
        t = fn()
        sk.set_tensor_block_pass(False)
        f = fn()
    finally:
        sk.set_tensor_block_pass(prev)
    return t, f


@pytest.mark.parametrize("d,n,m,ell", [(2, 3000, 2500, 24), (1, 2100, 2049, 16), (3, 2047, 2300, 32),
                                        (4, 2500, 1800, 5), (2, 4096, 4096, 32),
                                        # work units of 2 output tiles x 2 input blocks (plan_i8)
                                        (2, 30000, 12000, 12)])
def test_tensor_block_pass_matches_fp64_and_oracle(d, n, m, ell):
    rng, x, y, a, b = _points(d, n, m, d * 7919 + n + ell)
    eps = 0.02
    gp = sk.PointProblem(x, y, a, b, eps)
    op = O.Instance(a, b, eps, x=x, y=y)
    f = rng.uniform(-0.05, 0.05, n)
    g = O.ctransform_of_f(op, f)
    V = np.asfortranarray(rng.standard_normal((n, ell)))
    basis = sk.SpectralBasis(V, V, np.zeros(ell), eps)
    (gt, Ht), (gf, Hf) = _both_paths(lambda: sk.restricted_derivatives(gp, f, basis, g))
    go, Ho = O.restricted_derivatives(op, f, g, V)
    assert rel_err(gt, go) <= 1e-9 and rel_err(Ht, Ho) <= 1e-11
    assert rel_err(gf, go) <= 1e-9 and rel_err(Hf, Ho) <= 1e-11
    # the two device paths: same grad to the FP64 pass's own agreement with the oracle
    assert rel_err(Ht, Hf) <= 1e-12


def test_tensor_block_pass_sknr_solve_matches_fp64_and_oracle():
    """C4-shaped (uniform square, eps = 5e-4 scaled to n) SK-NR(16) solve with a smooth
    basis: identical iteration counts and accept decisions on both device paths and
    against the oracle (stable accept test), potentials within 1e-9."""
    inst = G.config("C4", n=2048, m=2048)
    eps = 4e-3
    gp = sk.PointProblem(inst.x, inst.y, inst.alpha, inst.beta, eps, inst.cost_scale)
    op = O.Instance(inst.alpha, inst.beta, eps, x=inst.x, y=inst.y, cost_div=1.0 / inst.cost_scale)
    V = np.asfortranarray(smooth_basis(inst.x, inst.alpha, 16))
    basis = sk.SpectralBasis(V, V, np.zeros(16), eps)

    def run():
        return sk.solve(gp, tol=1e-9, max_iter=3000, ell=16, basis=basis, trace=True, accept="stable")

    rt, rf = _both_paths(run)
    with O.accept_mode("stable"):
        ro = O.solve(op, tol=1e-9, max_iter=3000, ell=16, V=V, trace=True)
    assert rt.converged and rf.converged and ro["converged"]
    assert rt.iterations == rf.iterations == ro["iterations"]
    acc_t = [t.newton_accepted for t in rt.trace]
    acc_o = [bool(t[4]) for t in ro["trace"]]
    assert acc_t == [t.newton_accepted for t in rf.trace] == acc_o
    assert rel_err(rt.f, ro["f"]) <= 1e-9 and rel_err(rt.g, ro["g"]) <= 1e-9


def test_basis_digit_tiles_follow_the_solve():
    """The basis' int8 digit tiles are made once per solve (prepare_solve) and reused by every
    Newton pass of that solve; a second solve on the same handle with another basis, and a
    restricted_derivatives call in between (its own W), must not see stale tiles."""
    inst = G.config("C4", n=2048, m=2048)
    eps = 4e-3
    rng = np.random.default_rng(5)
    Va = np.asfortranarray(smooth_basis(inst.x, inst.alpha, 8))
    Vb = np.asfortranarray(np.linalg.qr(rng.standard_normal((2048, 8)))[0] * np.sqrt(2048.0))
    ba = sk.SpectralBasis(Va, Va, np.zeros(8), eps)
    bb = sk.SpectralBasis(Vb, Vb, np.zeros(8), eps)

    def make():
        return sk.PointProblem(inst.x, inst.y, inst.alpha, inst.beta, eps, inst.cost_scale)

    def run(p, basis):
        return sk.solve(p, tol=1e-9, max_iter=40, ell=8, basis=basis, trace=True, accept="stable")

    p = make()
    ra = run(p, ba)
    f0 = rng.uniform(-0.01, 0.01, 2048)
    sk.restricted_derivatives(p, f0, bb)
    rb = run(p, bb)
    ra2 = run(p, ba)
    rb_fresh = run(make(), bb)
    assert np.array_equal(rb.f, rb_fresh.f) and np.array_equal(rb.g, rb_fresh.g)
    assert np.array_equal(ra.f, ra2.f) and ra.iterations == ra2.iterations
    assert [t.newton_accepted for t in rb.trace] == [t.newton_accepted for t in rb_fresh.trace]
