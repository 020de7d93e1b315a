"""Portable seeded generator, restating the reference's `parorb::Rng`
(include/parorb/rng.hpp:13-41): std::mt19937_64 with an explicit
53-bit bits->double conversion and Box-Muller normals with a spare.

Used host-side for the synthetic problem geometry (atom placement, charges,
Gaussian-well centres) — a few thousand draws. Bulk orbital normals come from
the native library (`po_rng_normals`), which restates the same generator in
C++ so both produce the reference's exact bits for a seed.
"""
from __future__ import annotations

import math

_MASK64 = (1 << 64) - 1


class Rng:
    """mt19937_64 + `uniform()` / `uniform(lo, hi)` / `normal()` as in rng.hpp."""

    def __init__(self, seed: int):
        mt = [0] * 312
        mt[0] = seed & _MASK64
        for i in range(1, 312):
            mt[i] = (6364136223846793005 * (mt[i - 1] ^ (mt[i - 1] >> 62)) + i) & _MASK64
        self._mt = mt
        self._idx = 312
        self._spare = 0.0
        self._have_spare = False

    def _twist(self) -> None:
        mt = self._mt
        for i in range(312):
            x = (mt[i] & 0xFFFFFFFF80000000) | (mt[(i + 1) % 312] & 0x7FFFFFFF)
            xa = x >> 1
            if x & 1:
                xa ^= 0xB5026F5AA96619E9
            mt[i] = mt[(i + 156) % 312] ^ xa
        self._idx = 0

    def next_u64(self) -> int:
        if self._idx >= 312:
            self._twist()
        y = self._mt[self._idx]
        self._idx += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & _MASK64

    def uniform(self, lo: float | None = None, hi: float | None = None) -> float:
        u = float(self.next_u64() >> 11) * 2.0 ** -53
        if lo is None:
            return u
        return lo + (hi - lo) * u

    def normal(self) -> float:
        if self._have_spare:
            self._have_spare = False
            return self._spare
        u1 = self.uniform()
        while u1 == 0.0:
            u1 = self.uniform()
        r = math.sqrt(-2.0 * math.log(u1))
        theta = 2.0 * math.pi * self.uniform()
        self._spare = r * math.sin(theta)
        self._have_spare = True
        return r * math.cos(theta)
