"""Seeded xorshift64* streams, bit-identical to the reference generator.

Reference: /root/reference/pkg/src/ghostmg/rng.py:14-56 (splitmix64 seeding,
xorshift64* step, ``uniform() = (x >> 11) * 2**-53``, ``uniform_symmetric``).

The reference draws ``uniform_symmetric(n)`` with a Python loop, which is
unusable at 513^3 nodes.  Here the stream is cut into lanes; the start state
of each lane is obtained with a GF(2) jump-ahead (the xorshift state update is
linear over GF(2)), and all lanes then advance together with vectorised
uint64 arithmetic.  The draw order is the reference's stream order, so the
output is bit-for-bit the same sequence.
"""

import numpy as np

_MASK = (1 << 64) - 1
STAR = 2685821657736338717
_GOLDEN = 0x9E3779B97F4A7C15


def splitmix64(x):
    """(next_carry, mixed) for one splitmix64 step."""
    x = (x + _GOLDEN) & _MASK
    z = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & _MASK
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _MASK
    return x, z ^ (z >> 31)


def seed_state(seed):
    carry, state = splitmix64(int(seed) & _MASK)
    if state == 0:
        _, state = splitmix64(carry)
    return state


def _step(s):
    s ^= s >> 12
    s = (s ^ (s << 25)) & _MASK
    s ^= s >> 27
    return s


class XorShift64Star:
    """Scalar stream with the reference's interface."""

    def __init__(self, seed=42):
        self._state = seed_state(seed)

    def next_u64(self):
        self._state = _step(self._state)
        return (self._state * STAR) & _MASK

    def uniform(self):
        return (self.next_u64() >> 11) * (2.0 ** -53)

    def uniform_symmetric(self, n):
        out = _bulk_symmetric(self._state, int(n))
        # leave the scalar stream where the reference would
        self._state = _jump(self._state, int(n))
        return out


# ---- GF(2) jump-ahead ---------------------------------------------------
# A linear map on 64-bit states is stored as its 64 column images.

def _step_columns():
    return [_step(1 << b) for b in range(64)]


def _apply(cols, s):
    out = 0
    b = 0
    while s:
        if s & 1:
            out ^= cols[b]
        s >>= 1
        b += 1
    return out


def _compose(a, b):
    """Columns of a∘b (apply b first)."""
    return [_apply(a, c) for c in b]


def _power_columns(k):
    result = [1 << b for b in range(64)]
    base = _step_columns()
    while k:
        if k & 1:
            result = _compose(base, result)
        base = _compose(base, base)
        k >>= 1
    return result


def _jump(state, k):
    return _apply(_power_columns(k), state) if k else state


def _bulk_symmetric(state, n, lanes=4096):
    if n <= 0:
        return np.empty(0, dtype=np.float64)
    if n < 4 * lanes:
        out = np.empty(n, dtype=np.float64)
        s = state
        for i in range(n):
            s = _step(s)
            out[i] = 2.0 * ((((s * STAR) & _MASK) >> 11) * (2.0 ** -53)) - 1.0
        return out
    length = -(-n // lanes)
    jump = _power_columns(length)
    starts = np.empty(lanes, dtype=np.uint64)
    s = state
    for b in range(lanes):
        starts[b] = s
        s = _apply(jump, s)
    cur = starts.copy()
    block = np.empty((length, lanes), dtype=np.uint64)
    star = np.uint64(STAR)
    with np.errstate(over="ignore"):
        for i in range(length):
            cur ^= cur >> np.uint64(12)
            cur ^= cur << np.uint64(25)
            cur ^= cur >> np.uint64(27)
            block[i] = cur * star
    words = block.T.ravel()[:n]
    return 2.0 * ((words >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)) - 1.0


def uniform_symmetric(seed, n):
    """n draws from (-1, 1) of a fresh stream seeded with ``seed``."""
    return _bulk_symmetric(seed_state(seed), int(n))
