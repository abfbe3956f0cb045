"""Seeded fixtures with the reference's implementation-independent mappings (rng.hpp:15-32).

A tiny pure-Python std::mt19937_64 for the handful of draws config generation needs (segment
lengths); bulk tensor inputs are generated on the device.
"""
from __future__ import annotations

_MASK = (1 << 64) - 1


class MT19937_64:
    def __init__(self, seed: int):
        self.mt = [0] * 312
        self.mt[0] = seed & _MASK
        for i in range(1, 312):
            prev = self.mt[i - 1]
            self.mt[i] = (6364136223846793005 * (prev ^ (prev >> 62)) + i) & _MASK
        self.idx = 312

    def _twist(self):
        um, lm = 0xFFFFFFFF80000000, 0x7FFFFFFF
        mt = self.mt
        for i in range(312):
            x = (mt[i] & um) | (mt[(i + 1) % 312] & lm)
            xa = x >> 1
            if x & 1:
                xa ^= 0xB5026F5AA96619E9
            mt[i] = mt[(i + 156) % 312] ^ xa
        self.idx = 0

    def __call__(self) -> int:
        if self.idx >= 312:
            self._twist()
        x = self.mt[self.idx]
        self.idx += 1
        x ^= (x >> 29) & 0x5555555555555555
        x ^= (x << 17) & 0x71D67FFFEDA60000
        x ^= (x << 37) & 0xFFF7EEE000000000
        x ^= x >> 43
        return x & _MASK


def uniform_below(gen: MT19937_64, bound: int) -> int:
    """rng.hpp:25-32 (no modulo bias)."""
    limit = bound * (_MASK // bound)
    while True:
        draw = gen()
        if draw < limit:
            return draw % bound


def uniform_unit(gen: MT19937_64) -> float:
    """rng.hpp:15-17"""
    return (gen() >> 11) * 2.0 ** -53
