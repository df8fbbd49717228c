"""Pins for the FIFO and FIRO comparison buffers of oracle/reservoir.py
(reading R21 in DESIGN.md).

* FIFO, from its definition ("batched ... according to the order they are
  received", "seen once, and only once", "suspended when the FIFO buffer is
  full"): on random schedules every batch is the next B items in arrival order
  (put_seq consecutive), every accepted item is drawn exactly once by EOS, the
  population never exceeds C, a batch needs p >= B during reception.
* FIRO ("extracted from random positions", "evicted upon reading", threshold,
  "set to zero once data production is over"): exhaustive enumeration of every
  draw outcome shows that a batch of B from a list of p items is a uniformly
  random B-subset (each subset with probability 1 / C(p, B), a closed form), and
  that the remaining items are drained exactly once; the Philox-driven oracle
  matches the subset law statistically (chi^2); the gate is p >= theta + B.
"""
import random
from fractions import Fraction
from itertools import combinations
from math import comb

import numpy as np

from oracle.reservoir import EAGAIN, FIFO, FIRO, OK, Reservoir
from test_oracle_reservoir import enumerate_runs


def _put(res, i):
    return res.put(i, 0, np.zeros(5, np.float32), None)


def test_fifo_order_once_and_backpressure():
    for seed in range(20):
        rng = random.Random(seed)
        C = rng.randint(2, 9)
        B = rng.randint(1, min(4, C))                        # FIFO needs B <= C
        res = Reservoir(C, 0, 1, keep_payload=False, policy=FIFO)
        drawn, nxt, puts = [], 0, 0
        for _ in range(40):
            for _ in range(rng.randint(0, 5)):
                assert _put(res, puts) == OK
                puts += 1
            p_before = min(C, res.p + len(res.pend))          # after the commit point
            st, slots = res.sample(B)
            res.check_invariants()
            assert res.p <= C
            if p_before < B:
                assert st == EAGAIN and slots == []
                continue
            assert st == OK and len(slots) == B
            seqs = [int(res.put_seq[j]) for j in slots]
            assert seqs == list(range(nxt, nxt + B)), (seqs, nxt)
            nxt += B
            drawn += [int(res.sim[j]) for j in slots]
        res.close()
        while True:
            st, slots = res.sample(B)
            res.check_invariants()
            assert st == OK
            if not slots:
                break
            assert len(slots) <= B
            drawn += [int(res.sim[j]) for j in slots]
        assert drawn == list(range(puts)), "every item exactly once, in arrival order"
        assert res.hist[1] == puts and res.hist.sum() == puts


def test_fifo_suspends_production_when_full():
    res = Reservoir(3, 0, 1, keep_payload=False, policy=FIFO)
    for i in range(5):
        _put(res, i)
    st, slots = res.sample(1)
    assert st == OK and [int(res.sim[j]) for j in slots] == [0]
    assert res.p == 2 and len(res.pend) == 2                 # 3 committed, 2 waiting
    st, slots = res.sample(3)                                 # commit fills to 3 again
    assert [int(res.sim[j]) for j in slots] == [1, 2, 3] and len(res.pend) == 1


def _firo_first_batch(p, B, theta):
    def run(chooser):
        res = Reservoir(p, theta, 1, chooser=chooser, keep_payload=False, policy=FIRO)
        for i in range(p):
            _put(res, i)
        st, slots = res.sample(B)
        assert st == OK
        first = tuple(sorted(int(res.sim[j]) for j in slots))
        res.close()
        rest = []
        while True:
            st, s = res.sample(B)
            if not s:
                break
            rest += [int(res.sim[j]) for j in s]
        res.check_invariants()
        assert sorted(list(first) + rest) == list(range(p)), "each item exactly once"
        return first
    return run


def test_firo_batch_is_uniform_subset_exhaustive():
    for p, B in ((4, 2), (5, 3), (3, 1)):
        runs = enumerate_runs(_firo_first_batch(p, B, theta=0))
        assert sum(w for w, _ in runs) == 1
        dist = {}
        for w, first in runs:
            dist[first] = dist.get(first, Fraction(0)) + w
        assert set(dist) == set(combinations(range(p), B))
        assert all(v == Fraction(1, comb(p, B)) for v in dist.values())


def test_firo_philox_subset_chi2():
    p, B = 5, 2
    subsets = list(combinations(range(p), B))
    counts = dict.fromkeys(subsets, 0)
    n = 2000
    for seed in range(1, n + 1):
        res = Reservoir(p, 0, 1, seed=seed, keep_payload=False, policy=FIRO)
        for i in range(p):
            _put(res, i)
        _, slots = res.sample(B)
        counts[tuple(sorted(int(res.sim[j]) for j in slots))] += 1
    e = n / len(subsets)
    chi2 = sum((c - e) ** 2 / e for c in counts.values())
    assert chi2 < 27.88     # chi2(9), p = 0.001


def test_firo_gate_and_zero_threshold_after_close():
    res = Reservoir(10, 3, 1, keep_payload=False, policy=FIRO)
    for i in range(4):
        _put(res, i)
    assert res.sample(2)[0] == EAGAIN                          # 4 < theta + B = 5
    _put(res, 4)
    st, s = res.sample(2)                                      # draws see 5 and 4 items > 3
    assert st == OK and len(s) == 2 and res.p == 3
    assert res.sample(2)[0] == EAGAIN                          # 3 < 5
    res.close()                                                # threshold -> 0
    sizes = []
    while True:
        st, s = res.sample(2)
        if not s:
            break
        sizes.append(len(s))
    assert sizes == [2, 1] and res.p == 0
