"""Pins of oracle/dataset.py (the offline baseline's epoch order, reading R24)."""
import itertools
import math

import numpy as np

from oracle import dataset as od


def test_is_a_permutation_and_reproducible():
    for n in (0, 1, 2, 7, 1000):
        p = od.epoch_order(n, seed=9, epoch=3)
        assert sorted(p.tolist()) == list(range(n))
        assert np.array_equal(p, od.epoch_order(n, seed=9, epoch=3))
    assert not np.array_equal(od.epoch_order(1000, 9, 0), od.epoch_order(1000, 9, 1))
    assert not np.array_equal(od.epoch_order(1000, 9, 0), od.epoch_order(1000, 10, 0))


def test_draws_to_orders_is_a_bijection():
    """Fisher-Yates: the n! draw sequences (j_i in [0, i]) give the n! orders once each,
    so uniform draws give uniform orders (Knuth TAOCP 3.4.2, Algorithm P)."""
    for n in range(1, 6):
        seen = set()
        for js in itertools.product(*[range(i + 1) for i in range(n - 1, 0, -1)]):
            it = iter(js)
            p = tuple(od.epoch_order(n, 0, 0, chooser=lambda i: next(it)).tolist())
            seen.add(p)
        assert len(seen) == math.factorial(n)


def test_orders_are_uniform_over_seeds():
    """n = 3 over 6000 (seed, epoch) pairs: each of the 6 orders within 5 sigma of 1000."""
    counts = {}
    for s in range(600):
        for e in range(10):
            p = tuple(od.epoch_order(3, s, e).tolist())
            counts[p] = counts.get(p, 0) + 1
    assert len(counts) == 6
    sigma = math.sqrt(6000 * (1 / 6) * (5 / 6))
    assert all(abs(c - 1000) < 5 * sigma for c in counts.values()), counts


def test_batches_drop_the_partial_tail():
    b = od.batches(10, 3, seed=1, epoch=0)
    assert len(b) == 3 and all(len(x) == 3 for x in b)
    assert np.array_equal(np.concatenate(b), od.epoch_order(10, 1, 0)[:9])
