"""Seeded synthetic inputs for BASELINE.json configs C1-C5.

SplitMix64 exactly as the reference harness (proj/include/sknr/harness/rng.hpp:13-50):
uniform01 = (next_u64 >> 11) * 2^-53, uniform(lo,hi) = lo + (hi-lo)*u, normal = Marsaglia
polar with a cached spare. Source stream seeded s, target stream seeded
s ^ 0xD1B54A32D192ED03 (experiments.cpp:85); points drawn point by point,
coordinate by coordinate, weights from the same stream after all points.
Points are returned column-major (n x d), like harness::PointCloud.

SplitMix64 is counter based (draw t of seed s is mix(s + (t+1)*gamma)), so pure
uniform streams are generated vectorised; streams that interleave rejection
sampling (normals) run through the sequential generator below.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

GAMMA = 0x9E3779B97F4A7C15
TARGET_XOR = 0xD1B54A32D192ED03
_M64 = (1 << 64) - 1


def _mix(z: np.ndarray) -> np.ndarray:
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def splitmix_u64(seed: int, start: int, count: int) -> np.ndarray:
    """Draws start .. start+count-1 of the stream seeded `seed`."""
    t = np.arange(start + 1, start + count + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed & _M64) + t * np.uint64(GAMMA)
        return _mix(z)


def u64_to_unit(z: np.ndarray) -> np.ndarray:
    return (z >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


class SplitMix64:
    """Sequential SplitMix64 with the reference's uniform/normal semantics."""

    def __init__(self, seed: int):
        self.seed = seed & _M64
        self.t = 0
        self.have_spare = False
        self.spare = 0.0
        self._buf = np.empty(0)
        self._pos = 0

    def _refill(self, need: int = 4096):
        self._buf = u64_to_unit(splitmix_u64(self.seed, self.t, need))
        self._pos = 0

    def uniform01(self) -> float:
        if self._pos >= self._buf.size:
            self._refill()
        v = float(self._buf[self._pos])
        self._pos += 1
        self.t += 1
        return v

    def uniform(self, lo: float, hi: float) -> float:
        return lo + (hi - lo) * self.uniform01()

    def uniform_block(self, count: int, lo: float = 0.0, hi: float = 1.0) -> np.ndarray:
        """`count` consecutive uniform(lo,hi) draws (vectorised)."""
        # consume whatever is buffered first to keep the stream position exact
        out = np.empty(count)
        k = 0
        while k < count and self._pos < self._buf.size:
            out[k] = self.uniform(lo, hi)
            k += 1
        if k < count:
            u = u64_to_unit(splitmix_u64(self.seed, self.t, count - k))
            out[k:] = lo + (hi - lo) * u
            self.t += count - k
            self._buf = np.empty(0)
            self._pos = 0
        return out

    def normal(self) -> float:
        if self.have_spare:
            self.have_spare = False
            return self.spare
        while True:
            u = self.uniform(-1.0, 1.0)
            v = self.uniform(-1.0, 1.0)
            q = u * u + v * v
            if not (q >= 1.0 or q == 0.0):
                break
        scale = math.sqrt(-2.0 * math.log(q) / q)
        self.spare = v * scale
        self.have_spare = True
        return u * scale


@dataclass
class Instance:
    name: str
    x: np.ndarray  # n x d, column-major
    y: np.ndarray  # m x d
    alpha: np.ndarray
    beta: np.ndarray
    epsilon: float
    ell: int
    cost_scale: float = 1.0
    epsilons: tuple = ()
    basis_eps: float = 0.0

    @property
    def n(self):
        return self.x.shape[0]

    @property
    def m(self):
        return self.y.shape[0]


def _uniform_cloud(rng: SplitMix64, count: int, d: int, lo: float, hi: float) -> np.ndarray:
    flat = rng.uniform_block(count * d, lo, hi)  # point by point, coordinate by coordinate
    return np.asfortranarray(flat.reshape(count, d))


def _normal_cloud(rng: SplitMix64, count: int, d: int, scale: float = 1.0) -> np.ndarray:
    pts = np.empty((count, d))
    for i in range(count):
        for k in range(d):
            pts[i, k] = scale * rng.normal()
    return np.asfortranarray(pts)


def _dirichlet1(rng: SplitMix64, count: int) -> np.ndarray:
    u = rng.uniform_block(count)
    e = -np.log1p(-u)  # E = -log(1 - U), avoids log 0
    return e / e.sum()


def _uniform_weights(count: int) -> np.ndarray:
    return np.full(count, 1.0 / count)


def config(name: str, seed: int = 1, n: int | None = None, m: int | None = None) -> Instance:
    """BASELINE.json configs; n/m override sizes for small parity cases."""
    name = name.upper()
    src = SplitMix64(seed)
    tgt = SplitMix64(seed ^ TARGET_XOR)
    if name == "C1":
        n = n or 512
        m = m or n
        x = _uniform_cloud(src, n, 2, 0.0, 1.0)
        y = _uniform_cloud(tgt, m, 2, 0.0, 1.0)
        return Instance("C1", x, y, _uniform_weights(n), _uniform_weights(m), 1e-2, 10, basis_eps=2e-2)
    if name == "C2":
        n = n or 4096
        m = m or n
        pts = np.empty((n, 2))
        for i in range(n):
            comp = -1.0 if src.uniform01() < 0.5 else 1.0
            pts[i, 0] = comp + 0.3 * src.normal()
            pts[i, 1] = 0.3 * src.normal()
        x = np.asfortranarray(pts)
        y = _uniform_cloud(tgt, m, 2, -2.0, 2.0)
        # C = ||x-y||^2 / max_ij ||x-y||^2
        cmax = 0.0
        for lo in range(0, n, 1024):
            d = x[lo:lo + 1024, None, :] - y[None, :, :]
            cmax = max(cmax, float(np.max(np.einsum("ijk,ijk->ij", d, d))))
        eps_sched = (0.1, 0.05, 0.025, 0.0125, 0.00625, 0.003125, 0.0015625, 0.001)
        return Instance("C2", x, y, _uniform_weights(n), _uniform_weights(m), 1e-3, 16,
                        cost_scale=1.0 / cmax, epsilons=eps_sched)
    if name == "C3":
        n = n or 16384
        m = m or n
        x = _uniform_cloud(src, n, 3, 0.0, 1.0)
        a = _dirichlet1(src, n)
        y = _normal_cloud(tgt, m, 3)
        b = _dirichlet1(tgt, m)
        return Instance("C3", x, y, a, b, 1e-3, 20, basis_eps=2e-3)
    if name == "C4":
        n = n or 65536
        m = m or n
        x = _uniform_cloud(src, n, 2, 0.0, 1.0)
        y = _uniform_cloud(tgt, m, 2, 0.0, 1.0)
        return Instance("C4", x, y, _uniform_weights(n), _uniform_weights(m), 5e-4, 32, basis_eps=1e-3)
    if name == "C5":
        n = n or 32768
        m = m or 16384
        x = _normal_cloud(src, n, 64, 0.125)
        wa = src.uniform_block(n, 0.5, 1.5)
        y = _normal_cloud(tgt, m, 64, 0.125)
        wb = tgt.uniform_block(m, 0.5, 1.5)
        return Instance("C5", x, y, wa / wa.sum(), wb / wb.sum(), 1e-3, 24, basis_eps=2e-3)
    raise ValueError(f"unknown config {name}")


def sq_euclidean_cost(x: np.ndarray, y: np.ndarray, cost_scale: float = 1.0) -> np.ndarray:
    """Dense C_ij = cost_scale * ||x_i - y_j||^2 in direct-difference form (generators.cpp:101)."""
    d = x[:, None, :] - y[None, :, :]
    c = np.einsum("ijk,ijk->ij", d, d)
    if cost_scale != 1.0:
        c = c / (1.0 / cost_scale)
    return np.asfortranarray(c)


# ---------------------------------------------------------------- named 2-d families
# harness generators (generators.cpp:19-92) and make_instance (experiments.cpp:83-106),
# used by the CLI's --synthetic flag. Points come back n x 2 column-major with
# uniform weights, drawn in the reference's order from the scalar stream.
def gaussian_cloud(count: int, mean, cov, seed: int):
    """mean + L z with L = chol(cov), z = (normal, normal) per point (generators.cpp:19-36)."""
    if count < 1:
        raise ValueError("gaussian_cloud: count must be positive")
    cov = np.asarray(cov, dtype=np.float64).reshape(2, 2)
    mean = np.asarray(mean, dtype=np.float64).reshape(2)
    if np.max(np.abs(cov - cov.T)) > 1e-12:
        raise ValueError("gaussian_cloud: covariance must be symmetric")
    # Eigen LLT of a 2 x 2 (lower factor)
    if not cov[0, 0] > 0.0:
        raise ValueError("gaussian_cloud: covariance must be positive definite")
    l00 = math.sqrt(cov[0, 0])
    l10 = cov[1, 0] / l00
    piv = cov[1, 1] - l10 * l10
    if not piv > 0.0:
        raise ValueError("gaussian_cloud: covariance must be positive definite")
    l11 = math.sqrt(piv)
    rng = SplitMix64(seed)
    pts = np.empty((count, 2))
    for i in range(count):
        z0 = rng.normal()
        z1 = rng.normal()
        pts[i, 0] = mean[0] + l00 * z0
        pts[i, 1] = mean[1] + (l10 * z0 + l11 * z1)
    return np.asfortranarray(pts), _uniform_weights(count)


def two_moons(count_per_moon: int, noise: float, seed: int):
    """Upper and lower half-moons (generators.cpp:38-59)."""
    if count_per_moon < 1:
        raise ValueError("two_moons: count must be positive")
    if noise < 0.0:
        raise ValueError("two_moons: noise must be nonnegative")
    rng = SplitMix64(seed)
    upper = np.empty((count_per_moon, 2))
    lower = np.empty((count_per_moon, 2))
    for i in range(count_per_moon):
        th = rng.uniform(0.0, math.pi)
        upper[i, 0] = math.cos(th) + noise * rng.normal()
        upper[i, 1] = math.sin(th) + noise * rng.normal()
    for i in range(count_per_moon):
        th = rng.uniform(0.0, math.pi)
        lower[i, 0] = 1.0 - math.cos(th) + noise * rng.normal()
        lower[i, 1] = 0.5 - math.sin(th) + noise * rng.normal()
    w = _uniform_weights(count_per_moon)
    return (np.asfortranarray(upper), w), (np.asfortranarray(lower), w.copy())


def annulus_and_square(count_annulus: int, count_square: int, r_in: float, r_out: float, side: float,
                       seed: int):
    """Rejection-sampled annulus and a uniform square from one stream (generators.cpp:61-92)."""
    if count_annulus < 1 or count_square < 1:
        raise ValueError("annulus_and_square: counts must be positive")
    if not (0.0 <= r_in < r_out):
        raise ValueError("annulus_and_square: need 0 <= r_in < r_out")
    if not side > 0.0:
        raise ValueError("annulus_and_square: side must be positive")
    rng = SplitMix64(seed)
    ann = np.empty((count_annulus, 2))
    for i in range(count_annulus):
        while True:
            x = rng.uniform(-r_out, r_out)
            y = rng.uniform(-r_out, r_out)
            q = x * x + y * y
            if not (q > r_out * r_out or q < r_in * r_in):
                break
        ann[i] = (x, y)
    half = side / 2.0
    sq = np.empty((count_square, 2))
    for i in range(count_square):
        sq[i, 0] = rng.uniform(-half, half)
        sq[i, 1] = rng.uniform(-half, half)
    return ((np.asfortranarray(ann), _uniform_weights(count_annulus)),
            (np.asfortranarray(sq), _uniform_weights(count_square)))


def make_instance(family: str, n: int, m: int, seed: int = 1, noise: float = 0.05, r_in: float = 0.5,
                  r_out: float = 1.0, side: float = 2.0):
    """(x, alpha, y, beta) of a named family (experiments.cpp:83-106): gauss2d | two_moons |
    annulus_square; target stream seeded seed ^ 0xD1B54A32D192ED03."""
    tseed = (seed ^ TARGET_XOR) & _M64
    if family == "gauss2d":
        xs, a = gaussian_cloud(n, (0.0, 0.0), np.eye(2), seed)
        yt, b = gaussian_cloud(m, (4.0, 4.0), [[1.0, -0.8], [-0.8, 1.0]], tseed)
        return xs, a, yt, b
    if family == "two_moons":
        (xs, a), _ = two_moons(n, noise, seed)
        _, (yt, b) = two_moons(m, noise, tseed)
        return xs, a, yt, b
    if family == "annulus_square":
        (xs, a), (yt, b) = annulus_and_square(n, m, r_in, r_out, side, seed)
        return xs, a, yt, b
    raise ValueError(f"make_instance: unknown family '{family}'")
