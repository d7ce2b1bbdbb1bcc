"""Bit-exact host restatement of the reference's batch sampling RNG:
``std::mt19937_64`` and libstdc++'s ``std::uniform_int_distribution<size_t>``
(train.cpp:387-404 draws ``samples[pick(rng)]`` per batch item).

The training loop needs the same (camera, frame) schedule as the reference
for the same seed, so the generator is restated exactly (pinned against the
oracle's C++ draws in tests/test_rng.py).  Host-side integer work: a few draws
per iteration.
"""
from __future__ import annotations

_MASK64 = (1 << 64) - 1


class MT19937_64:
    """std::mt19937_64 (the 64-bit Mersenne Twister of [rand.predef])."""

    _N, _M = 312, 156
    _MATRIX_A = 0xB5026F5AA96619E9
    _UPPER, _LOWER = 0xFFFFFFFF80000000, 0x7FFFFFFF

    def __init__(self, seed: int = 5489):
        self.mt = [0] * self._N
        self.mt[0] = seed & _MASK64
        for i in range(1, self._N):
            self.mt[i] = (6364136223846793005 * (self.mt[i - 1] ^ (self.mt[i - 1] >> 62)) + i) & _MASK64
        self.idx = self._N

    def _twist(self) -> None:
        mt, N, M = self.mt, self._N, self._M
        for i in range(N):
            x = (mt[i] & self._UPPER) | (mt[(i + 1) % N] & self._LOWER)
            xa = x >> 1
            if x & 1:
                xa ^= self._MATRIX_A
            mt[i] = mt[(i + M) % N] ^ xa
        self.idx = 0

    def __call__(self) -> int:
        if self.idx >= self._N:
            self._twist()
        y = self.mt[self.idx]
        self.idx += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & _MASK64


def uniform_index(g: MT19937_64, lo: int, hi: int) -> int:
    """std::uniform_int_distribution<size_t>(lo, hi)(g) as libstdc++ (GCC >= 11)
    computes it for a full 64-bit generator: Lemire's nearly divisionless
    multiply-shift on 128-bit products (bits/uniform_int_dist.h, _S_nd)."""
    urange = hi - lo
    if urange == _MASK64:
        return g()
    erange = urange + 1
    product = g() * erange
    low = product & _MASK64
    if low < erange:
        threshold = ((-erange) & _MASK64) % erange
        while low < threshold:
            product = g() * erange
            low = product & _MASK64
    return lo + (product >> 64)


def generate_canonical(g: MT19937_64) -> float:
    """std::generate_canonical<double, 53>(g) for a 64-bit engine (libstdc++:
    one draw, converted to double, divided by 2^64, clamped below 1)."""
    r = float(g()) / 18446744073709551616.0
    return r if r < 1.0 else 0.9999999999999999


class NormalDistribution:
    """std::normal_distribution<double>(0, 1) as libstdc++ implements it: the
    Marsaglia polar method, the second variate of each pair cached in the
    distribution object (so the reference's draw order matters)."""

    def __init__(self):
        self.saved = None

    def __call__(self, g: MT19937_64) -> float:
        import math

        if self.saved is not None:
            v, self.saved = self.saved, None
            return v
        while True:
            x = 2.0 * generate_canonical(g) - 1.0
            y = 2.0 * generate_canonical(g) - 1.0
            r2 = x * x + y * y
            if r2 <= 1.0 and r2 != 0.0:
                break
        mult = math.sqrt(-2.0 * math.log(r2) / r2)
        self.saved = x * mult
        return y * mult


def densify_normals(g: MT19937_64, kinds3, kinds4):
    """The normal variates densify_and_prune (train.cpp:182-299) draws, in its
    order, laid out for hgs_densify_apply: statics -- a fresh distribution
    per sample_normal3 (train.cpp:68-72), 6 doubles per densified Gaussian
    (clone: one triple, split: two); dynamics -- ONE distribution for the pool,
    Vec4(nd, nd, nd, nd) built from draws taken right to left (g++ argument
    order), 8 doubles per densified Gaussian (clone: one Vec4, split: two)."""
    import numpy as np

    n3 = np.zeros(6 * max(1, len(kinds3)))
    for r, k in enumerate(kinds3):
        for h in range(1 if k == 1 else 2):
            nd = NormalDistribution()
            n3[6 * r + 3 * h: 6 * r + 3 * h + 3] = [nd(g), nd(g), nd(g)]
    n4 = np.zeros(8 * max(1, len(kinds4)))
    nd = NormalDistribution()
    for r, k in enumerate(kinds4):
        for h in range(1 if k == 1 else 2):
            d0, d1, d2, d3 = nd(g), nd(g), nd(g), nd(g)
            n4[8 * r + 4 * h: 8 * r + 4 * h + 4] = [d3, d2, d1, d0]
    return n3, n4
