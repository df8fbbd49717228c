"""ORACLE (test infrastructure only -- never imported by the product path).

Counter-based RNG used by every stochastic component of the method ("All
the stochastic components ... are seeded"; the paper does not name a generator,
reading Q8 in DESIGN.md fixes Philox4x32-10).

Philox4x32-10 as published by Salmon, Moraes, Dror, Shaw, "Parallel random
numbers: as easy as 1, 2, 3", SC'11 (Random123): multipliers 0xD2511F53 and
0xCD9E8D57, Weyl key increments 0x9E3779B9 and 0xBB67AE85, 10 rounds.

Stream layout:
  key     = (lo32(seed), hi32(seed))
  counter = (lo32(n), hi32(n), c2, tag)
  r64     = (o1 << 32) | o0                        (words o2, o3 unused)
  bounded(n) = floor(r64 * n / 2^64)                (no rejection)
  unit       = (r64 >> 11) * 2^-53                  (double in [0, 1))
Pins: tests/golden/philox_kat.txt (Random123 known-answer vectors),
tests/test_oracle_philox.py (bounded() preimage counts by brute force).
"""
from __future__ import annotations

import numpy as np

M0 = 0xD2511F53
M1 = 0xCD9E8D57
W0 = 0x9E3779B9
W1 = 0xBB67AE85
MASK32 = 0xFFFFFFFF

# stream tags (counter word 3)
TAG_SAMPLE = 1
TAG_EVICT = 2
TAG_DRAIN = 3
TAG_INIT = 4
TAG_EPOCH = 5     # offline baseline epoch order (reading R24)


def philox4x32_10(ctr, key):
    """Vectorised Philox4x32-10.  ctr: 4 arrays (or ints) of uint32 words,
    key: 2 words.  Returns 4 uint64 arrays holding 32-bit outputs."""
    c0, c1, c2, c3 = (np.asarray(c, dtype=np.uint64) & np.uint64(MASK32) for c in ctr)
    k0 = np.asarray(key[0], dtype=np.uint64) & np.uint64(MASK32)
    k1 = np.asarray(key[1], dtype=np.uint64) & np.uint64(MASK32)
    m32 = np.uint64(MASK32)
    for rnd in range(10):
        if rnd > 0:
            k0 = (k0 + np.uint64(W0)) & m32
            k1 = (k1 + np.uint64(W1)) & m32
        p0 = np.uint64(M0) * c0          # < 2^64, exact in uint64
        p1 = np.uint64(M1) * c2
        hi0, lo0 = p0 >> np.uint64(32), p0 & m32
        hi1, lo1 = p1 >> np.uint64(32), p1 & m32
        c0, c1, c2, c3 = (hi1 ^ c1 ^ k0), lo1, (hi0 ^ c3 ^ k1), lo0
    return c0, c1, c2, c3


def r64(seed: int, tag: int, n, c2):
    """One 64-bit draw per counter value n (array or int)."""
    n = np.asarray(n, dtype=np.uint64)
    key = (seed & MASK32, (seed >> 32) & MASK32)
    o0, o1, _, _ = philox4x32_10((n & np.uint64(MASK32), n >> np.uint64(32),
                                  np.full_like(n, c2), np.full_like(n, tag)), key)
    return (o1 << np.uint64(32)) | o0


def bounded(r, n):
    """floor(r * n / 2^64) for uint64 r and 0 <= n < 2^32, computed exactly with
    32-bit halves (no overflow: see the bound in DESIGN.md)."""
    r = np.asarray(r, dtype=np.uint64)
    n = np.uint64(n)
    rh, rl = r >> np.uint64(32), r & np.uint64(MASK32)
    return (rh * n + ((rl * n) >> np.uint64(32))) >> np.uint64(32)


def unit_double(r):
    r = np.asarray(r, dtype=np.uint64)
    return (r >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def draw_index(seed: int, tag: int, n_ctr: int, c2: int, pop: int) -> int:
    """Scalar helper: bounded(r64(seed, tag, n_ctr, c2), pop)."""
    return int(bounded(r64(seed, tag, n_ctr, c2), pop))
