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
