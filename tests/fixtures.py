"""Seeded test fixtures restated from the reference's tests.

* ``Rng`` — flowroi::Rng (/root/reference/proj/include/flowroi/rng.hpp:11-62): splitmix64 with a
  0x9e3779b97f4a7c15 seed xor and two warm-up draws, Box–Muller normals caching the spare.
* ``textured_frame``, ``random_frame``, ``cyclic_shift``, ``random_mask`` —
  testutil (/root/reference/proj/tests/test_util.hpp:37-76).

``math`` uses the platform libm, the same one the reference links, so these produce the same
samples as the C++ fixtures (pinned in tests/test_oracle_pin.py against golden vectors).
"""
from __future__ import annotations

import math

import numpy as np

M64 = (1 << 64) - 1


class Rng:
    def __init__(self, seed: int):
        self.state = (seed ^ 0x9E3779B97F4A7C15) & M64
        self.have_spare = False
        self.spare = 0.0
        self.next_u64()
        self.next_u64()

    def next_u64(self) -> int:
        self.state = (self.state + 0x9E3779B97F4A7C15) & M64
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
        return z ^ (z >> 31)

    def next_double(self) -> float:
        return float(self.next_u64() >> 11) * (2.0 ** -53)

    def uniform(self, lo: float, hi: float) -> float:
        return lo + (hi - lo) * self.next_double()

    def next_below(self, n: int) -> int:
        return self.next_u64() % n

    def normal(self, mean: float = 0.0, sigma: float = 1.0) -> float:
        return mean + sigma * self._std_normal()

    def _std_normal(self) -> float:
        if self.have_spare:
            self.have_spare = False
            return self.spare
        u1 = 0.0
        while u1 <= 0.0:
            u1 = self.next_double()
        u2 = self.next_double()
        r = math.sqrt(-2.0 * math.log(u1))
        a = 6.283185307179586476925286766559 * u2
        self.spare = r * math.sin(a)
        self.have_spare = True
        return r * math.cos(a)


def clamp_to_depth(v: float, depth: int) -> int:
    """core.hpp:148-152 (std::lround: half away from zero)."""
    maxval = float((1 << depth) - 1)
    v = 0.0 if v < 0.0 else v
    v = maxval if maxval < v else v
    return int(math.floor(v + 0.5)) if v - math.floor(v) != 0.5 else int(math.floor(v)) + 1


def textured_frame(w: int, h: int, depth: int, seed: int, noise_sigma: float = 12.0) -> np.ndarray:
    rng = Rng(seed)
    maxval = (1 << depth) - 1
    unit = maxval / 255.0
    out = np.empty((h, w), np.uint16)
    for y in range(h):
        cy = math.cos(2.0 * 3.14159265358979 * y / 31.0)
        for x in range(w):
            v = (0.35 * maxval + 28.0 * unit * math.sin(2.0 * 3.14159265358979 * x / 37.0) * cy
                 + rng.normal(0.0, noise_sigma * unit))
            out[y, x] = clamp_to_depth(v, depth)
    return out


def random_frame(w: int, h: int, depth: int, seed: int) -> np.ndarray:
    rng = Rng(seed)
    maxval = (1 << depth) - 1
    return np.array([rng.next_u64() & maxval for _ in range(w * h)], np.uint16).reshape(h, w)


def cyclic_shift(f: np.ndarray, dx: int, dy: int) -> np.ndarray:
    """out(x, y) = f((x - dx) mod w, (y - dy) mod h)."""
    return np.roll(f, (dy, dx), axis=(0, 1)).copy()


def random_mask(w: int, h: int, fill: float, seed: int) -> np.ndarray:
    rng = Rng(seed)
    return np.array([1 if rng.next_double() < fill else 0 for _ in range(w * h)],
                    np.uint8).reshape(h, w)
