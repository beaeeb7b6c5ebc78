"""Random small instances restated from the reference's test helpers
(T/helpers.hpp:13-50) so the GPU box can regenerate the golden corpora
without /root/reference. Test infrastructure only.

InstanceRng wraps std::mt19937_64; `pick(lo, hi)` = lo + gen() % (hi-lo+1).
random_stream / random_episode draw in exactly the reference's order, which
the golden fixture pins per instance with an FNV-1a digest of the stream.
"""
from __future__ import annotations

MASK64 = (1 << 64) - 1


class MT19937_64:
    """std::mt19937_64 (the C++ standard's parameters)."""
    N, M = 312, 156
    A = 0xB5026F5AA96619E9
    UPPER, LOWER = 0xFFFFFFFF80000000, 0x7FFFFFFF

    def __init__(self, seed: int):
        mt = [0] * self.N
        mt[0] = seed & MASK64
        for i in range(1, self.N):
            mt[i] = (6364136223846793005 * (mt[i - 1] ^ (mt[i - 1] >> 62)) + i) & MASK64
        self.mt = mt
        self.idx = self.N

    def _twist(self):
        mt, N, M, A = self.mt, self.N, self.M, self.A
        for i in range(N):
            x = (mt[i] & self.UPPER) | (mt[(i + 1) % N] & self.LOWER)
            xa = x >> 1
            if x & 1:
                xa ^= A
            mt[i] = mt[(i + M) % N] ^ xa
        self.idx = 0

    def __call__(self) -> int:
        if self.idx >= self.N:
            self._twist()
        y = self.mt[self.idx]
        self.idx += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & MASK64


class InstanceRng:
    def __init__(self, seed: int):
        self.gen = MT19937_64(seed)

    def pick(self, lo: int, hi: int) -> int:
        return lo + self.gen() % (hi - lo + 1)


POOL = [(0, 5), (5, 10), (2, 7)]


def random_stream(rng: InstanceRng, max_events=200, max_alphabet=6, max_gap=3):
    n = rng.pick(0, max_events)
    alphabet = rng.pick(1, max_alphabet)
    types, times = [], []
    t = 0
    for _ in range(n):
        t += rng.pick(0, max_gap)
        types.append(rng.pick(0, alphabet - 1))
        times.append(t)
    return types, times, alphabet


def random_episode(rng: InstanceRng, alphabet: int, max_size=4):
    n = rng.pick(1, max_size)
    types, cons = [], []
    for i in range(n):
        types.append(rng.pick(0, alphabet - 1))
        if i > 0:
            cons.append(POOL[rng.pick(0, 2)])
    return types, cons


def fnv_stream(types, times, alphabet) -> str:
    h = 1469598103934665603

    def mix(v):
        nonlocal h
        for b in range(8):
            h ^= (v >> (8 * b)) & 0xFF
            h = (h * 1099511628211) & MASK64

    mix(len(types))
    mix(alphabet)
    for ty, tm in zip(types, times):
        mix(ty)
        mix(tm & MASK64)
    return f"{h:016x}"


def corpus(seed, count, max_events=200, max_alphabet=6, max_gap=3, max_size=4):
    """Yields (types, times, alphabet, ep_types, constraints) like the
    reference test loops."""
    rng = InstanceRng(seed)
    for _ in range(count):
        types, times, a = random_stream(rng, max_events, max_alphabet, max_gap)
        et, cons = random_episode(rng, a, max_size)
        yield types, times, a, et, cons
