"""Pins for oracle/reservoir.py (Algorithm 1).

* Brute force: the worked example in tests/golden/reservoir_worked_example.txt
  was derived by hand from the algorithm text:
    SAMPLE(2) commits a,b (p=2 > theta=1) and draws (0,0),(0,1),(1,0),(1,1).
    SAMPLE(1)'s commit appends c, then d must evict a *seen* item:
      (2,0): only a is seen -> a (seen 2) evicted, u becomes C so e stays pending;
      (0,2): symmetric -> b (seen 2);
      (1,1): r-th seen of {a, b} uniform -> (a,1) or (b,1); e then evicts the other.
    e is pending with prob 1/2; at CLOSE it evicts the one item SAMPLE(1) marked,
    uniform over the 3 live items -> second victim (a,1) 1/12+1/4 = 1/3, (b,1) 1/3,
    (c,1) 1/6, (d,1) 1/6.  Every path retires a/b, then drains 3 items:
    hist {1:4, 2:1}, drain sizes 2, 1, 0.
  The exhaustive enumerator below runs the oracle's code under every random
  outcome with exact Fraction weights and must reproduce these rationals; the
  Philox-driven oracle must match them statistically (chi^2).
* Closed form: the Appendix residency law p(k) = (1/n)(1-1/n)^k, mean n-1
  (P:537-548), in the regime where every item is seen before the next put.
* Invariants after every op on random schedules (no unseen loss P:279, eviction
  of seen only P:268, conservation S:191, bounds, never-blocks-after-threshold
  P:279), plus the blocking examples S:162-182.
"""
import os
import random
from fractions import Fraction

import numpy as np
import pytest

from oracle import philox
from oracle.reservoir import EAGAIN, ECLOSED, EPROTO, OK, Reservoir

GOLD = os.path.join(os.path.dirname(__file__), "golden", "reservoir_worked_example.txt")


class NeedChoice(Exception):
    def __init__(self, n):
        self.n = n


def enumerate_runs(run):
    """Exhaustively enumerate every outcome of run(chooser) with exact weights."""
    results = []
    stack = [([], Fraction(1))]
    while stack:
        prefix, prob = stack.pop()
        it = iter(prefix)

        def chooser(tag, ctr, n):
            try:
                c = next(it)
            except StopIteration:
                raise NeedChoice(n)
            return c
        try:
            results.append((prob, run(chooser)))
        except NeedChoice as e:
            for c in range(e.n):
                stack.append((prefix + [c], prob / e.n))
    return results


NAMES = "abcde"


def worked_example(chooser=None, seed=1):
    res = Reservoir(3, 1, 1, seed=seed, chooser=chooser, keep_payload=False)
    out = {"victims": [], "drain": []}

    def put(i):
        res.put(i, 0, np.zeros(5, np.float32), None)

    def victims_since(k):
        for (_, j, esim, et, eseen) in res.commit_log[k:]:
            if esim >= 0:
                out["victims"].append((NAMES[esim], eseen))

    put(0); put(1)
    k = len(res.commit_log); st, _ = res.sample(2); victims_since(k)
    assert st == OK
    put(2); put(3); put(4)
    k = len(res.commit_log); res.sample(1); victims_since(k)
    out["e_pending"] = len(res.pend) == 1
    k = len(res.commit_log); res.close(); victims_since(k)
    for _ in range(3):
        st, s = res.sample(2)
        out["drain"].append(len(s))
        res.check_invariants()
    out["evictions"] = res.evictions
    out["hist"] = {i: int(v) for i, v in enumerate(res.hist) if v}
    return out


def _golden():
    g = {}
    for line in open(GOLD):
        if line.startswith("#") or not line.strip():
            continue
        key, val, prob = line.split()
        g.setdefault(key, {})[val] = Fraction(prob)
    return g


def test_worked_example_exhaustive_enumeration():
    g = _golden()
    runs = enumerate_runs(worked_example)
    assert sum(p for p, _ in runs) == 1
    dist = {}
    for p, o in runs:
        fv = "(%s,%d)" % o["victims"][0]
        sv = "(%s,%d)" % o["victims"][1]
        for key, val in (("first_victim", fv), ("second_victim", sv),
                         ("e_pending_after_sample1", "yes" if o["e_pending"] else None),
                         ("evictions", str(o["evictions"])),
                         ("hist", "{" + ",".join("%d:%d" % kv for kv in sorted(o["hist"].items())) + "}"),
                         ("drain_sizes", ",".join(map(str, o["drain"])))):
            if val is not None:
                dist.setdefault(key, {}).setdefault(val, Fraction(0))
                dist[key][val] += p
    assert dist["first_victim"] == g["first_victim"]
    assert dist["second_victim"] == g["second_victim"]
    assert dist["e_pending_after_sample1"] == g["e_pending_after_sample1"]
    assert dist["evictions"] == g["evictions"]
    assert dist["hist"] == g["hist"]
    assert dist["drain_sizes"] == g["drain_sizes"]


def test_worked_example_philox_frequencies_chi2():
    g = _golden()["first_victim"]
    keys = sorted(g)
    counts = dict.fromkeys(keys, 0)
    n = 3000
    for seed in range(1, n + 1):
        o = worked_example(seed=seed)
        counts["(%s,%d)" % o["victims"][0]] += 1
    chi2 = sum((counts[k] - n * float(g[k])) ** 2 / (n * float(g[k])) for k in keys)
    assert chi2 < 16.27   # chi2(3), p = 0.001


def _random_schedule(seed, C, theta, B, steps, puts_max):
    rng = random.Random(seed)
    res = Reservoir(C, theta, 4, seed=seed, keep_payload=True)
    sim = 0
    seen_once = set()
    evicted_unseen = 0
    for _ in range(steps):
        for _ in range(rng.randrange(puts_max + 1)):
            res.put(sim, 0, np.zeros(5, np.float32), np.full(4, 100.0 + sim, np.float32))
            sim += 1
        k = len(res.commit_log)
        st, slots = res.sample(rng.randrange(1, B + 1))
        for (_, j, esim, et, eseen) in res.commit_log[k:]:
            if esim >= 0 and eseen == 0:
                evicted_unseen += 1
        for j in slots:
            seen_once.add(int(res.sim[j]))
        res.check_invariants()
    res.close()
    res.check_invariants()
    while True:
        st, slots = res.sample(B)
        res.check_invariants()
        if not slots:
            break
    return res, evicted_unseen, sim


@pytest.mark.parametrize("seed", range(8))
def test_invariants_random_schedules(seed):
    res, evicted_unseen, n_put = _random_schedule(seed, C=24, theta=5, B=6, steps=120, puts_max=4)
    assert evicted_unseen == 0                      # P:279 "avoiding discarding any unseen data"
    assert res.q == n_put and res.p == 0 and res.over
    assert int(np.sum(res.hist)) == n_put           # every committed item retired exactly once
    assert res.d == int(np.sum(np.arange(len(res.hist)) * res.hist))   # S:191 conservation


def test_put_blocks_when_all_unseen_and_get_blocks_below_threshold():
    res = Reservoir(3, 1, 1, keep_payload=False)
    for i in range(5):
        res.put(i, 0, np.zeros(5, np.float32), None)
    res.commit()
    assert res.p == 3 and len(res.pend) == 2        # put waits while not_seen == C
    r2 = Reservoir(1001, 1000, 1, keep_payload=False)
    for i in range(1000):
        r2.put(i, 0, np.zeros(5, np.float32), None)
    assert r2.sample(10)[0] == EAGAIN               # p = theta blocks
    r2.put(1000, 0, np.zeros(5, np.float32), None)
    assert r2.sample(10)[0] == OK


def test_protocol_errors_and_drain_examples():
    res = Reservoir(4, 0, 1, keep_payload=False)
    res.put(0, 0, np.zeros(5, np.float32), None)
    assert res.close() == OK
    assert res.close() == EPROTO                    # S:178 double signal
    assert res.put(1, 0, np.zeros(5, np.float32), None) == ECLOSED
    st, s = res.sample(3)
    assert st == OK and s == [0]                    # S:182 exactly one more get
    st, s = res.sample(3)
    assert st == OK and s == []                     # then end-of-stream
    empty = Reservoir(4, 2, 1, keep_payload=False)
    empty.close()
    assert empty.sample(1) == (OK, [])              # S:181 empty + signal -> EOS


def test_consumer_never_blocks_after_threshold_under_stalled_production():
    res = Reservoir(50, 10, 1, keep_payload=False)
    for i in range(11):
        res.put(i, 0, np.zeros(5, np.float32), None)
    for _ in range(200):                             # production stalls
        st, s = res.sample(8)
        assert st == OK and len(s) == 8


def test_residency_law_appendix():
    # with uniform eviction over n items the residency (number of later
    # inserts survived) is geometric, p(k) = (1/n)(1-1/n)^k, mean n-1.  The
    # Reservoir evicts uniformly over *seen* items, so test where all are seen:
    # a batch of 400 draws between puts leaves an item unseen w.p. (63/64)^400.
    n, m, B = 64, 12000, 400
    res = Reservoir(n, 0, 1, seed=11, keep_payload=False)
    born, life = {}, []
    for i in range(m):
        k = len(res.commit_log)
        res.put(i, 0, np.zeros(5, np.float32), None)
        res.sample(B)
        for (qq, j, esim, et, eseen) in res.commit_log[k:]:
            born[qq] = i
            if esim >= 0:
                life.append(i - born[esim] - 1)   # sim id == put index == put_seq here
    life = np.array(life[n:])
    assert abs(life.mean() - (n - 1)) < 0.05 * (n - 1)
    # shape: P(k=0) = 1/n within a generous tolerance
    assert abs(np.mean(life == 0) - 1 / n) < 0.01


def test_paper_like_stream_repeat_statistics():
    # P:337-343 (Fig. 3): most samples are seen "a couple of times", rarely up to ~8.
    C, theta, B = 600, 100, 10
    res = Reservoir(C, theta, 1, seed=5, keep_payload=False)
    rng = random.Random(1)
    puts = 0
    while puts < 2500:
        for _ in range(7 if rng.random() < 0.5 else 8):   # ~0.75 puts per draw
            res.put(puts, 0, np.zeros(5, np.float32), None); puts += 1
        for _ in range(1):
            res.sample(B)
    res.close()
    while res.sample(B)[1]:
        pass
    h = res.hist
    assert h[0] == 0                     # nothing retired unseen
    assert np.argmax(h) == 1             # mode at one occurrence
    assert 1.0 < res.d / res.q < 3.0
