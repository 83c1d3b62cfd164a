"""Fixtures mirroring the reference's tests/support.hpp:14-101 (SplitMix64 seeded)."""
import numpy as np

from paper_2506_14780_b200.generators import SplitMix64


def random_measure(rng: SplitMix64, size: int) -> np.ndarray:
    w = np.array([0.2 + rng.uniform01() for _ in range(size)])
    return w / w.sum()


def random_problem_data(rng: SplitMix64, n: int, m: int, cost_scale: float = 2.0):
    """(cost, alpha, beta) of support.hpp:21-28: cost filled column by column."""
    cost = np.empty((n, m), order="F")
    for j in range(m):
        for i in range(n):
            cost[i, j] = cost_scale * rng.uniform01()
    a = random_measure(rng, n)
    b = random_measure(rng, m)
    return cost, a, b


def random_vector(rng: SplitMix64, size: int, scale: float = 1.0) -> np.ndarray:
    return np.array([scale * rng.uniform(-1.0, 1.0) for _ in range(size)])


def symmetric_2x2():
    cost = np.array([[0.0, 1.0], [1.0, 0.0]], order="F")
    half = np.array([0.5, 0.5])
    return cost, half, half


def symmetric_2x2_optimum(eps=1.0):
    g = -eps * np.log(0.5 * (1.0 + np.exp(-1.0 / eps)))
    return np.zeros(2), np.full(2, g)


def gauge_normalized(alpha, f, g):
    c = float(np.dot(alpha, f))
    return f - c, g + c


def rel_err(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    scale = max(np.max(np.abs(b)), 1e-300)
    return float(np.max(np.abs(a - b)) / scale)


def projector_distance(A, B):
    """||P_A - P_B||_2 for orthonormal column blocks (spectral.cpp:232-244)."""
    R = B - A @ (A.T @ B)
    return float(min(1.0, np.linalg.svd(R, compute_uv=False).max()))


def smooth_basis(x, alpha, ell):
    """ell low-frequency cosine modes of a 2-D projection of the sources, orthonormal in
    L2(alpha) and alpha-mean-zero (the deflated direction removed): a Newton basis whose
    steps are large and well decided, with no top_modes run needed on either side."""
    rng = np.random.default_rng(0)
    z = x @ rng.standard_normal((x.shape[1], 2))
    z = (z - z.min(0)) / (z.max(0) - z.min(0))
    cols = [np.cos(np.pi * a * z[:, 0]) * np.cos(np.pi * b * z[:, 1])
            for a in range(8) for b in range(8) if (a, b) != (0, 0)]
    w = np.sqrt(alpha)[:, None]
    Vs = np.stack(cols[:ell], 1) * w
    Vs -= w * (w[:, 0] @ Vs)[None, :]
    Q, _ = np.linalg.qr(Vs)
    return np.asfortranarray(Q / w)
