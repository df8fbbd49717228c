"""Pins for oracle/philox.py: published known-answer vectors and brute-force
properties of the bounded-integer mapping."""
import os
import random

import numpy as np
import pytest

from oracle import philox

GOLD = os.path.join(os.path.dirname(__file__), "golden", "philox_kat.txt")


def _kat():
    for line in open(GOLD):
        if line.startswith("#") or not line.strip():
            continue
        w = [int(x, 16) for x in line.split()]
        yield w[0:4], w[4:6], w[6:10]


@pytest.mark.parametrize("ctr,key,want", list(_kat()))
def test_philox_known_answers(ctr, key, want):
    got = [int(x) for x in philox.philox4x32_10(ctr, key)]
    assert got == want


def test_philox_vectorised_equals_scalar():
    n = np.arange(1000, 1100, dtype=np.uint64)
    vec = philox.r64(12345678901, philox.TAG_SAMPLE, n, 3)
    for i, c in enumerate(range(1000, 1100)):
        o = philox.philox4x32_10((c, 0, 3, philox.TAG_SAMPLE), (12345678901 & 0xFFFFFFFF, 12345678901 >> 32))
        assert int(vec[i]) == (int(o[1]) << 32) | int(o[0])


def test_bounded_matches_exact_integer_arithmetic():
    rng = random.Random(7)
    cases = [(0, 1), (2**64 - 1, 2**32 - 1), (2**64 - 1, 1), (2**63, 6000), (1, 2**32 - 1)]
    cases += [(rng.getrandbits(64), rng.randrange(1, 2**32)) for _ in range(2000)]
    for r, n in cases:
        assert int(philox.bounded(np.uint64(r), n)) == (r * n) >> 64


@pytest.mark.parametrize("n", [1, 2, 3, 5, 7, 48, 200, 1000, 6000, 65535])
def test_bounded_preimage_counts_exhaustive_16bit(n):
    # r = k * 2^48 exercises the 16-bit analog floor(k*n/2^16) through the 64-bit
    # code path; every outcome must have floor or ceil(2^16/n) preimages.
    k = np.arange(2**16, dtype=np.uint64) << np.uint64(48)
    out = philox.bounded(k, n).astype(np.int64)
    assert out.min() == 0 and out.max() == n - 1
    counts = np.bincount(out, minlength=n)
    lo, hi = (2**16) // n, -(-(2**16) // n)
    assert set(np.unique(counts)) <= {lo, hi}


def test_unit_double_range_and_uniformity():
    u = philox.unit_double(philox.r64(1, philox.TAG_INIT, np.arange(200000, dtype=np.uint64), 0))
    assert u.min() >= 0.0 and u.max() < 1.0
    hist = np.histogram(u, bins=20, range=(0, 1))[0]
    exp = len(u) / 20
    chi2 = float(np.sum((hist - exp) ** 2 / exp))
    assert chi2 < 43.8  # chi2(19) p=0.001
