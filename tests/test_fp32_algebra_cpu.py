"""CPU checks of the fp32 variant's arithmetic (pts_f32_kernel),
emulated in numpy float32: the re-expansion around the squared distance is the same
exponent as the fp64 pack, the potential terms on the 2^-8 grid add exactly in fp32,
and at C4 scales the per-term error is a few 1e-6 and does not depend on the
potentials (a fixed perturbation of the kernel)."""
import numpy as np

from paper_2506_14780_b200 import generators as G

LS = 256.0 / np.log(2.0)  # 1/256-bit units per nat
INV_SQRT512 = 1.0 / np.sqrt(512.0)


def packs(x, y, f, g, eps):
    """fp64 packs as k_prep_in / k_prep_out build them (centred coordinates, u in 1/256 bits)."""
    c = 0.5 * (np.minimum(x.min(0), y.min(0)) + np.maximum(x.max(0), y.max(0)))
    xc, yc = x - c, y - c
    sigma = np.sqrt(2.0 * LS / eps)
    A = LS * (np.log(1.0 / len(x)) + f / eps - (xc ** 2).sum(1) / eps)
    B = LS * (g / eps - (yc ** 2).sum(1) / eps)
    return A, sigma * xc, B, sigma * yc


def f32_terms(A, X, B, Y):
    """2^v per cell with the fp32 kernel's rounding (v = u/256 in log2 units)."""
    Ap = A + 0.5 * (X ** 2).sum(1)
    Bp = B + 0.5 * (Y ** 2).sum(1)
    Ah, Bh = np.rint(Ap), np.rint(Bp)
    w = np.exp2((Ap - Ah) / 256.0).astype(np.float32)
    bs = np.exp2((Bp - Bh) / 256.0)
    Ahf = (Ah / 256.0).astype(np.float32)
    Bhf = (Bh / 256.0).astype(np.float32)
    Xs = (X * INV_SQRT512).astype(np.float32)
    Ys = (Y * INV_SQRT512).astype(np.float32)
    d = Xs[:, None, :] - Ys[None, :, :]
    q = (d[..., 0] * d[..., 0]).astype(np.float32)
    for k in range(1, X.shape[1]):
        q = (q + d[..., k] * d[..., k]).astype(np.float32)
    s = (Ahf[:, None] + Bhf[None, :]).astype(np.float32)
    v = (s - q).astype(np.float32)
    return w[:, None].astype(np.float64) * np.exp2(v.astype(np.float64)) * bs[None, :], s, Ahf, Bhf


def test_reexpansion_is_the_same_exponent():
    r = np.random.default_rng(0)
    A, B = r.normal(0, 1e5, 50), r.normal(0, 1e5, 40)
    X, Y = r.normal(0, 300, (50, 2)), r.normal(0, 300, (40, 2))
    u = A[:, None] + B[None, :] + X @ Y.T
    Ap, Bp = A + 0.5 * (X ** 2).sum(1), B + 0.5 * (Y ** 2).sum(1)
    u2 = Ap[:, None] + Bp[None, :] - 0.5 * ((X[:, None, :] - Y[None, :, :]) ** 2).sum(-1)
    assert np.max(np.abs(u - u2)) <= 1e-9 * np.max(np.abs(Ap))


def test_grid_sums_are_exact_in_fp32():
    r = np.random.default_rng(1)
    ah = np.rint(r.uniform(-2 ** 22, 2 ** 22, 10000)) / 256.0  # |.| < 2^14
    bh = np.rint(r.uniform(-2 ** 22, 2 ** 22, 10000)) / 256.0
    s32 = (ah.astype(np.float32) + bh.astype(np.float32)).astype(np.float64)
    assert np.array_equal(s32, ah + bh)


def test_c4_scale_terms_are_a_fixed_perturbation():
    inst = G.config("C4", n=2000, m=300)
    eps = inst.epsilon
    # smooth (c-concave-like) potentials as the solver produces them, not noise: the
    # terms that carry each column are then at short distance
    f = 0.05 * np.sin(3.0 * inst.x[:, 0]) * np.cos(2.0 * inst.x[:, 1])
    g0 = np.zeros(inst.m)
    # terms near the column maximum carry the sum: compare those
    A, X, B, Y = packs(inst.x, inst.y, f, g0, eps)
    u = A[:, None] + B[None, :] + X @ Y.T
    B = B - u.max(0)  # exact shift: max term 1 per column
    u = A[:, None] + B[None, :] + X @ Y.T
    exact = np.exp2(u / 256.0)
    t32, _, _, _ = f32_terms(A, X, B, Y)
    big = exact > 1e-6
    rel = np.abs(t32[big] - exact[big]) / exact[big]
    assert rel.max() < 5e-5
    cols = np.abs(t32.sum(0) - exact.sum(0)) / exact.sum(0)
    assert cols.max() < 2e-5
    # moving the potentials by an arbitrary amount changes the rounding of Ah, Bh but not
    # the per-term error of the terms: the perturbation depends on the coordinates only
    shift = 0.37 * LS  # a third of a nat, absorbed by A and B in opposite directions
    t32b, _, _, _ = f32_terms(A + shift, X, B - shift, Y)
    assert np.max(np.abs(t32b[big] - t32[big]) / t32[big]) < 2e-7
