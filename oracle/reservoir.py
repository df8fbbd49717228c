"""ORACLE (test infrastructure only -- never imported by the product path).

The Reservoir training buffer of the paper, Algorithm 1 and
its prose, in the canonical deterministic form fixed by DESIGN.md
readings R1-R7 (readings Q1-Q9):

  PUT(item):  if closed -> ECLOSED.  pend.push_back(item)          (Alg.1 put)
  COMMIT():   while pend not empty:
                 if u == C: break            # P:264 "Block until one element gets seen"
                 item = pend.pop_front()
                 if p < C: j = p; p += 1     # fill phase (dense prefix)
                 else:                       # P:267-269 "Evict one seen element"
                    r = bounded_EVICT(q)(s); j = r-th slot (ascending id) with seen > 0
                    hist[seen[j]] += 1; evictions += 1
                 slot[j] = item; seen[j] = 0; put_seq[j] = q; q += 1
              if closed and pend empty: over = true
  SAMPLE(B):  COMMIT()
              if not over:
                 if p <= theta: return EAGAIN
                 i_b = bounded_SAMPLE(d+b)(p) for b < B
                 seen[i_b] += 1 for every draw; d += B                # P:250 unseen->seen
              else:  drain ("until it finally empties out"):
                 repeat B times while p > 0:
                    k = bounded_DRAIN(d)(p); d += 1; j = pos[k]
                    seen[j] += 1; hist[seen[j]] += 1; out.append(j)
                    pos[k] = pos[p-1]; p -= 1
  CLOSE():    if closed -> EPROTO.  closed = true; COMMIT()

The two comparison buffers of P:221-223 share the put / pending / commit-point
machinery (reading R21):
  FIFO: COMMIT appends while p < C at slot (h + p) mod C (a ring; a full buffer
        suspends production = puts stay pending).  SAMPLE(B) takes the B oldest
        items (slots h..h+B-1 mod C) and removes them; during reception it needs
        p >= B ("as soon as the buffer can provide one"), after close it returns
        min(B, p).  Each item is seen exactly once.
  FIRO: COMMIT appends while p < C at list position p (slot pos[p]).  SAMPLE(B)
        makes B draws, each k = bounded_DRAIN(d)(p) over the current list with
        removal (swap with the last position); during reception every one of the
        B draws must see more than theta items, i.e. p >= theta + B; the
        threshold is 0 after close ("set to zero once data production is over").

Stored payload (reading R8, P:210 fp32 wire data, normalisation reading Q13):
  F32 storage : RN_f32((u_f32 - 100f) / 400f)
  BF16 storage: RNE_bf16(RN_f32((u_f32 - 100f) / 400f))
Each random choice goes through `self.choose(tag, counter, n)` so the same code
can be driven by Philox (the method) or by an exhaustive enumerator (the pin in
tests/test_oracle_reservoir.py).
"""
from __future__ import annotations

from collections import deque

import numpy as np

from . import philox

OK, EAGAIN, ECLOSED, EPROTO = 0, 1, -2, -3
RESERVOIR, FIFO, FIRO = 0, 1, 2
HIST_BINS = 64

STORE_F32, STORE_BF16 = 0, 1


def normalise_f32(u_f32: np.ndarray) -> np.ndarray:
    """RN_f32((u - 100f) / 400f), each op an IEEE fp32 op (numpy float32)."""
    u = np.asarray(u_f32, dtype=np.float32)
    return (u - np.float32(100.0)) / np.float32(400.0)


def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even fp32 -> bf16, returned as uint16 bit patterns
    (finite inputs).  Written from the IEEE definition: keep the top 16 bits,
    add half an ulp minus one plus the lsb of the kept part (ties to even)."""
    b = np.asarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    lsb = (b >> np.uint64(16)) & np.uint64(1)
    return ((b + np.uint64(0x7FFF) + lsb) >> np.uint64(16)).astype(np.uint16)


def bf16_bits_to_f64(h: np.ndarray) -> np.ndarray:
    return (np.asarray(h, dtype=np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32).astype(np.float64)


def stored_payload(field_f32: np.ndarray, storage: int) -> np.ndarray:
    tn = normalise_f32(field_f32)
    return tn if storage == STORE_F32 else f32_to_bf16_bits(tn)


def stored_to_f64(payload: np.ndarray, storage: int) -> np.ndarray:
    if storage == STORE_F32:
        return np.asarray(payload, dtype=np.float32).astype(np.float64)
    return bf16_bits_to_f64(payload)


class Reservoir:
    """One rank's Reservoir.  Items are (sim, t, X[5] fp32, field fp32[N])."""

    def __init__(self, capacity: int, threshold: int, n_field: int, seed: int = 1,
                 rank: int = 0, storage: int = STORE_F32, chooser=None, keep_payload=True,
                 policy: int = RESERVOIR):
        if not (0 <= threshold < capacity):
            raise ValueError("require 0 <= threshold < capacity (P:321 uses 1000 < 6000)")
        self.C, self.theta, self.N = capacity, threshold, n_field
        self.policy = policy
        self.h = 0                      # FIFO ring head
        self.seed, self.rank, self.storage = seed, rank, storage
        self.keep_payload = keep_payload
        self.choose = chooser if chooser is not None else self._philox_choose
        self._vector_draws = chooser is None
        C = capacity
        self.sim = np.full(C, -1, dtype=np.int64)
        self.t = np.full(C, -1, dtype=np.int64)
        self.X = np.zeros((C, 5), dtype=np.float32)
        self.seen = np.zeros(C, dtype=np.int64)
        self.put_seq = np.full(C, -1, dtype=np.int64)
        dt = np.float32 if storage == STORE_F32 else np.uint16
        self.payload = np.zeros((C, n_field), dtype=dt) if keep_payload else None
        self.pos = np.arange(C, dtype=np.int64)
        self.hist = np.zeros(HIST_BINS, dtype=np.int64)
        self.p = self.q = self.d = 0
        self.u = 0
        self.evictions = 0
        self.accepted = 0
        self.closed = self.over = False
        self.pend: deque = deque()
        self.ever_open = False        # p > theta has been reached during reception
        self.commit_log: list = []     # (put_seq, slot, evictee_sim, evictee_t, evictee_seen)

    # -- randomness -----------------------------------------------------------------
    def _philox_choose(self, tag: int, ctr: int, n: int) -> int:
        return philox.draw_index(self.seed, tag, ctr, self.rank, n)

    # -- Alg. 1 put ---------------------------------------------------------------------
    def put(self, sim: int, t: int, X, field) -> int:
        if self.closed:
            return ECLOSED
        self.pend.append((int(sim), int(t), np.asarray(X, dtype=np.float32).copy(),
                          None if field is None else np.asarray(field, dtype=np.float32)))
        self.accepted += 1
        return OK

    def _rank_select_seen(self, r: int) -> int:
        idx = np.flatnonzero(self.seen[: self.C] > 0)   # ascending slot id (p == C here)
        return int(idx[r])

    def commit(self) -> None:
        if self.policy != RESERVOIR:
            self._commit_queue()
            return
        C = self.C
        while self.pend:
            if self.u == C:
                break
            sim, t, X, field = self.pend.popleft()
            ev = (-1, -1, 0)
            if self.p < C:
                j = self.p
                self.p += 1
            else:
                s = self.p - self.u
                r = self.choose(philox.TAG_EVICT, self.q, s)
                j = self._rank_select_seen(r)
                ev = (int(self.sim[j]), int(self.t[j]), int(self.seen[j]))
                self.hist[min(int(self.seen[j]), HIST_BINS - 1)] += 1
                self.evictions += 1     # evictee is seen, so u only gains the new item
            self.sim[j], self.t[j] = sim, t
            self.X[j] = X
            if self.keep_payload and field is not None:
                self.payload[j] = stored_payload(field, self.storage)
            self.seen[j] = 0
            self.put_seq[j] = self.q
            self.commit_log.append((self.q, j) + ev)
            self.q += 1
            self.u += 1
        if self.closed and not self.pend:
            self.over = True

    # -- FIFO / FIRO --------------------------------------------------------
    def _commit_queue(self) -> None:
        C = self.C
        while self.pend and self.p < C:                   # full buffer: production suspended
            sim, t, X, field = self.pend.popleft()
            j = (self.h + self.p) % C if self.policy == FIFO else int(self.pos[self.p])
            self.p += 1
            self.sim[j], self.t[j] = sim, t
            self.X[j] = X
            if self.keep_payload and field is not None:
                self.payload[j] = stored_payload(field, self.storage)
            self.seen[j] = 0
            self.put_seq[j] = self.q
            self.commit_log.append((self.q, j, -1, -1, 0))
            self.q += 1
            self.u += 1
        if self.closed and not self.pend:
            self.over = True

    def _retire(self, j: int) -> None:
        self.seen[j] += 1                                 # seen once, then removed
        self.hist[min(int(self.seen[j]), HIST_BINS - 1)] += 1
        self.u -= 1

    def _sample_queue(self, B: int):
        need = (B if self.policy == FIFO else self.theta + B) if not self.over else 1
        if self.p < need:
            return EAGAIN, []
        n = min(B, self.p)
        out = []
        if self.policy == FIFO:
            for b in range(n):
                j = (self.h + b) % self.C
                self._retire(j)
                out.append(j)
            self.h = (self.h + n) % self.C
            self.p -= n
            self.d += n
            return OK, out
        for _ in range(n):
            k = self.choose(philox.TAG_DRAIN, self.d, self.p)
            self.d += 1
            j = int(self.pos[k])
            self._retire(j)
            out.append(j)
            self.pos[k], self.pos[self.p - 1] = self.pos[self.p - 1], j   # freed slot -> position p-1
            self.p -= 1
        return OK, out

    # -- Alg. 1 get (batch-atomic) -----------------------------------------------------
    def sample(self, B: int):
        """Returns (status, slots).  status EAGAIN during reception while p <= theta
        (Reservoir), p < B (FIFO), p < theta + B (FIRO)."""
        if self.policy != RESERVOIR:
            self.commit()
            if self.over and self.p == 0:
                return OK, []
            return self._sample_queue(B)
        self.commit()
        if not self.over:
            if self.p <= self.theta:
                assert not self.ever_open, "consumption locked after threshold passed (P:279)"
                return EAGAIN, []
            self.ever_open = True
            if self._vector_draws:
                n = np.arange(self.d, self.d + B, dtype=np.uint64)
                idx = philox.bounded(philox.r64(self.seed, philox.TAG_SAMPLE, n, self.rank), self.p)
                slots = [int(v) for v in idx]
            else:
                slots = [self.choose(philox.TAG_SAMPLE, self.d + b, self.p) for b in range(B)]
            idx = np.asarray(slots, dtype=np.int64)
            uniq = np.unique(idx)
            self.u -= int(np.sum(self.seen[uniq] == 0))      # 0 -> 1 transitions
            np.add.at(self.seen, idx, 1)                      # duplicates count twice (Q9)
            self.d += B
            return OK, slots
        out = []
        while len(out) < B and self.p > 0:
            k = self.choose(philox.TAG_DRAIN, self.d, self.p)
            self.d += 1
            j = int(self.pos[k])
            if self.seen[j] == 0:
                self.u -= 1
            self.seen[j] += 1
            self.hist[min(int(self.seen[j]), HIST_BINS - 1)] += 1
            out.append(j)
            self.pos[k] = self.pos[self.p - 1]
            self.p -= 1
        return OK, out

    def close(self) -> int:
        if self.closed:
            return EPROTO
        self.closed = True
        self.commit()
        return OK

    # -- observability --------------------------------------------------------------------
    def live_slots(self) -> np.ndarray:
        if self.policy == FIFO:
            return np.sort((self.h + np.arange(self.p)) % self.C)
        if self.policy == FIRO:
            return np.sort(self.pos[: self.p])
        return np.sort(self.pos[: self.p]) if self.over else np.arange(self.p)

    def stats(self) -> dict:
        live = self.live_slots()
        u = int(np.sum(self.seen[live] == 0))
        return dict(population=self.p, unseen=u, seen=self.p - u, puts=self.accepted,
                    committed=self.q, draws=self.d, evictions=self.evictions,
                    pending=len(self.pend), hist=self.hist.copy())

    def check_invariants(self) -> None:
        C = self.C
        assert 0 <= self.p <= C
        live = self.live_slots()
        u = int(np.sum(self.seen[live] == 0))
        assert u == self.u, (u, self.u)
        assert self.u <= C
        if self.policy == RESERVOIR and not self.over:
            assert np.array_equal(self.pos, np.arange(C)), "pos must be identity in reception"
        if self.policy != RESERVOIR:
            assert self.u == self.p, "FIFO / FIRO items are removed when seen"
            assert sorted(self.pos.tolist()) == list(range(C)), "pos is a permutation"
        # conservation: draws = sum k*hist + sum live seen, once nothing saturates
        if self.hist[-1] == 0:
            assert self.d == int(np.sum(np.arange(HIST_BINS) * self.hist)) + int(np.sum(self.seen[live]))
        assert int(np.sum(self.hist)) + self.p == self.q
        assert self.q + len(self.pend) == self.accepted
