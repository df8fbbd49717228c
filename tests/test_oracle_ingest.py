"""Pins of oracle/ingest.py against what the paper and arithmetic fix (no GPU)."""
import itertools

import numpy as np
import pytest

from oracle import ingest as oi


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_route_is_round_robin_from_the_client_id(world):
    """a client's time steps go round robin over all ranks, the first one to a
    rank chosen by the client id: balanced within one message, consecutive steps on
    consecutive ranks, and different clients start on different ranks."""
    tau = 37
    for c in range(2 * world + 1):
        ranks = [oi.route(c, t, world) for t in range(tau)]
        counts = np.bincount(ranks, minlength=world)
        assert counts.max() - counts.min() <= 1
        assert ranks[0] == c % world
        assert all((ranks[t + 1] - ranks[t]) % world == 1 % world for t in range(tau - 1))
    assert len({oi.route(c, 0, world) for c in range(world)}) == world


def test_rank_streams_partition_the_sends():
    sends = [(c, t) for t in range(5) for c in range(3)] + [(1, 0), (1, 1)]   # a restart of client 1
    streams = oi.rank_streams(sends, 2)
    assert sorted(sum(streams, [])) == sorted(sends)
    for r, st in enumerate(streams):
        assert all(oi.route(c, t, 2) == r for c, t in st)
        # each rank sees the sends in global send order
        idx = [sends.index(k) for k in dict.fromkeys(st)]
        assert idx == sorted(idx)


def test_server_accept_brute_force_tiny():
    """every distinct key is kept exactly once, at the position of its first
    arrival; exhaustively over all arrival sequences of length <= 5 on 3 keys."""
    keys = [(0, 0), (0, 1), (1, 0)]
    for n in range(6):
        for seq in itertools.product(keys, repeat=n):
            kept = oi.server_accept(seq)
            assert len(kept) == len(set(kept)) == len(set(seq))
            firsts = sorted(set(seq), key=seq.index)
            assert kept == firsts


def test_restart_resends_are_discarded():
    """A client that dies after t = 0..4 and restarts from t = 0 delivers each step once."""
    sends = [(7, t) for t in range(5)] + [(7, t) for t in range(10)]
    for r, st in enumerate(oi.rank_streams(sends, 3)):
        assert oi.server_accept(st) == [(7, t) for t in range(10) if oi.route(7, t, 3) == r]


def test_to_wire_is_round_to_nearest_even():
    """P:210 fp64 -> fp32: exact values unchanged, ties to even, |x - f| <= ulp/2."""
    ulp = 2.0 ** -23
    x = np.array([1.0, 300.0, 1 + ulp / 2, 1 + 1.5 * ulp, 1 + 2.5 * ulp, -(1 + ulp / 2), 1 + 0.75 * ulp])
    f = oi.to_wire(x)
    assert f.dtype == np.float32
    assert list(f.astype(np.float64)) == [1.0, 300.0, 1.0, 1 + 2 * ulp, 1 + 2 * ulp, -1.0, 1 + ulp]
    rng = np.random.default_rng(3)
    y = rng.uniform(100.0, 500.0, 10000)
    g = oi.to_wire(y).astype(np.float64)
    half_ulp = np.spacing(oi.to_wire(y)).astype(np.float64) / 2
    assert np.all(np.abs(y - g) <= half_ulp)
