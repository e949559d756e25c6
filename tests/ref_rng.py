"""Deterministic generator of the reference (splitmix64 + Box-Muller).

Restates ``sgp::Rng`` (proj/include/sgp/common.hpp:45-97) so synthetic inputs
are reproducible bit-for-bit against the reference's own generator: same
seed -> same stream of u64 / uniform / normal / index draws.
"""
from __future__ import annotations

import math

import numpy as np

_MASK = (1 << 64) - 1
_GOLDEN = 0x9E3779B97F4A7C15


class Rng:
    """splitmix64 stream (common.hpp:47-55) with the reference's derived draws."""

    def __init__(self, seed: int):
        self.state = (seed & _MASK) or _GOLDEN
        self._spare = 0.0
        self._have_spare = False

    def next_u64(self) -> int:
        self.state = (self.state + _GOLDEN) & _MASK
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _MASK
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _MASK
        return z ^ (z >> 31)

    def next_uniform(self) -> float:
        """Uniform in (0, 1] (common.hpp:58-60)."""
        return (float(self.next_u64() >> 11) + 1.0) * 2.0 ** -53

    def next_normal(self) -> float:
        """Box-Muller, second member cached (common.hpp:64-76)."""
        if self._have_spare:
            self._have_spare = False
            return self._spare
        u1 = self.next_uniform()
        u2 = self.next_uniform()
        r = math.sqrt(-2.0 * math.log(u1))
        a = 6.283185307179586476925286766559 * u2
        self._spare = r * math.sin(a)
        self._have_spare = True
        return r * math.cos(a)

    def next_index(self, n: int) -> int:
        """Uniform integer in [0, n) without modulo bias (common.hpp:79-84)."""
        limit = _MASK - (_MASK % n)
        v = self.next_u64()
        while v >= limit:
            v = self.next_u64()
        return v % n

    def normal_matrix(self, rows: int, cols: int) -> np.ndarray:
        """Row-major visiting order, column-major storage (common.hpp:86-91)."""
        out = np.empty((rows, cols), order="F")
        for i in range(rows):
            for j in range(cols):
                out[i, j] = self.next_normal()
        return out

    def uniform_matrix(self, rows: int, cols: int, lo: float, hi: float) -> np.ndarray:
        """random_matrix() of proj/tests/test_kernels.cpp:10-15."""
        out = np.empty((rows, cols), order="F")
        for i in range(rows):
            for j in range(cols):
                out[i, j] = lo + (hi - lo) * self.next_uniform()
        return out
