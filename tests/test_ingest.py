"""The ingest channel (include/mel_ingest.h) against oracle/ingest.py, on host cores:
separate client processes, shared-memory rings, routing, fp64 -> fp32 wire conversion,
the per-client restart log, back-pressure, and a client that dies mid-send."""
import os
import subprocess
import sys
import uuid

import numpy as np
import pytest

from mel_inputs import clients
from oracle import ingest as oi
from paper_2309_16743_b200 import mel

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLIENT = os.path.join(ROOT, "tests", "ingest_client.py")


@pytest.fixture(scope="module")
def lib():
    from paper_2309_16743_b200 import build
    build.build()
    return mel.load_library()


def _name():
    return "t" + uuid.uuid4().hex[:10]


def _spawn(name, world, client, t0, t1, n, finalize=False, env=None):
    cmd = [sys.executable, CLIENT, name, str(world), str(client), str(t0), str(t1), "--n-field", str(n)]
    if finalize:
        cmd.append("--finalize")
    return subprocess.Popen(cmd, env=dict(os.environ, **(env or {})))


def _drain(ing, until_eos=True, limit=10_000, timeout_us=20_000_000):
    got = []
    while len(got) < limit:
        st, m = ing.next(timeout_us)
        if st == mel.EOS or (st == mel.EAGAIN and not until_eos):
            break
        assert st == mel.OK, st
        got.append(m)
        ing.release()
    return got


def test_route_matches_the_oracle(lib):
    il = mel.load_ingest_library()
    for w in (1, 2, 3, 8):
        for c in range(10):
            for t in range(12):
                assert lib.mel_route(c, t, w) == il.mel_route(c, t, w) == oi.route(c, t, w)


def test_single_client_bit_exact_wire_and_metadata(lib):
    n, name = 1000, _name()
    ing = mel.Ingest(name, 0, n, slots=4, expected_clients=1)
    p = _spawn(name, 1, 5, 0, 9, n, finalize=True)
    got = _drain(ing)
    assert p.wait(60) == 0
    assert [(m["sim_id"], m["t"]) for m in got] == [(5, t) for t in range(9)]
    for m in got:
        ref = oi.to_wire(clients.client_field(5, m["t"], n))
        assert m["field"].tobytes() == ref.tobytes()
        assert m["X"].tobytes() == clients.client_X(5).tobytes()
    s = ing.stats()
    assert s["received"] == 9 and s["duplicates"] == 0 and s["finalized"] == 1 and s["bytes"] == 9 * 4 * n
    ing.destroy()


def test_restarted_client_resends_are_discarded(lib):
    """a client that disappears after t = 0..4 (no finalize) and restarts from
    t = 0 delivers every step once, on the rank the route gives."""
    n, name, world = 64, _name(), 2
    rings = [mel.Ingest(name, r, n, slots=16, expected_clients=1) for r in range(world)]
    assert _spawn(name, world, 3, 0, 5, n).wait(60) == 0
    assert _spawn(name, world, 3, 0, 10, n, finalize=True).wait(60) == 0
    sends = [(3, t) for t in range(5)] + [(3, t) for t in range(10)]
    for r, ing in enumerate(rings):
        got = [(m["sim_id"], m["t"]) for m in _drain(ing)]
        assert got == oi.server_accept(oi.rank_streams(sends, world)[r])
        assert ing.stats()["duplicates"] == sum(1 for t in range(5) if oi.route(3, t, world) == r)
        ing.destroy()


def test_many_clients_small_ring_backpressure(lib):
    """8 client processes, 2 ranks, 3-slot rings (every client waits for free slots):
    each rank receives exactly its routed keys, per-client order preserved, payloads
    bit-exact."""
    n, name, world, tau, nc = 256, _name(), 2, 25, 8
    rings = [mel.Ingest(name, r, n, slots=3, expected_clients=nc) for r in range(world)]
    procs = [_spawn(name, world, c, 0, tau, n, finalize=True) for c in range(nc)]
    got = [[] for _ in range(world)]
    done = [False] * world
    while not all(done):                       # one consumer thread serves both rings
        for r, ing in enumerate(rings):
            if done[r]:
                continue
            st, m = ing.next(1000)
            if st == mel.EOS:
                done[r] = True
            elif st == mel.OK:
                got[r].append(m)
                ing.release()
    assert all(p.wait(60) == 0 for p in procs)
    sends = [(c, t) for c in range(nc) for t in range(tau)]
    for r in range(world):
        keys = [(m["sim_id"], m["t"]) for m in got[r]]
        assert sorted(keys) == sorted(oi.rank_streams(sends, world)[r])
        for c in range(nc):
            ts = [t for cc, t in keys if cc == c]
            assert ts == sorted(ts)
        for m in got[r][::7]:
            assert m["field"].tobytes() == oi.to_wire(clients.client_field(m["sim_id"], m["t"], n)).tobytes()
        rings[r].destroy()


def test_client_dying_between_claim_and_publish_is_skipped(lib):
    """A claimed ticket whose client process is gone does not wedge the ring."""
    n, name = 32, _name()
    ing = mel.Ingest(name, 0, n, slots=8, expected_clients=1)
    assert _spawn(name, 1, 1, 0, 3, n, env={"MEL_INGEST_FAULT": "die_after_claim"}).wait(60) == 3
    assert _spawn(name, 1, 2, 0, 3, n, finalize=True).wait(60) == 0
    got = _drain(ing)
    assert [(m["sim_id"], m["t"]) for m in got] == [(2, t) for t in range(3)]
    assert ing.stats()["abandoned"] == 1
    ing.destroy()


def test_client_dying_between_reservation_and_ticket_does_not_wedge(lib):
    """A client killed after reserving a slot (pid written) but before taking the ticket:
    the next client takes the reservation over and the ring keeps flowing."""
    n, name = 32, _name()
    ing = mel.Ingest(name, 0, n, slots=8, expected_clients=1)
    assert _spawn(name, 1, 1, 0, 3, n, env={"MEL_INGEST_FAULT": "die_after_pid"}).wait(60) == 4
    assert _spawn(name, 1, 2, 0, 3, n, finalize=True).wait(60) == 0
    got = _drain(ing)
    assert [(m["sim_id"], m["t"]) for m in got] == [(2, t) for t in range(3)]
    assert ing.stats()["abandoned"] == 0
    ing.destroy()


def test_full_ring_and_protocol_errors(lib):
    n, name = 16, _name()
    ing = mel.Ingest(name, 0, n, slots=2)
    cl = mel.Client(name, 1, 0)
    f = np.zeros(n)
    X = np.zeros(5, np.float32)
    assert cl.send(0, X, f) == mel.OK and cl.send(1, X, f) == mel.OK
    assert cl.send(2, X, f, timeout_us=2000) == mel.EAGAIN          # no consumer: back-pressure
    st, m = ing.next(0)
    assert st == mel.OK and m["t"] == 0 and ing.outstanding() == 1
    assert cl.send(2, X, f, timeout_us=2000) == mel.EAGAIN          # returned but not released
    ing.release()
    assert cl.send(2, X, f, timeout_us=2000) == mel.OK
    assert ing.outstanding() == 0
    with pytest.raises(mel.MelError):
        ing.release()                                                # nothing outstanding
    assert [ing.next(0)[1]["t"] for _ in range(2)] == [1, 2]
    ing.release(); ing.release()
    assert cl.finalize(timeout_us=100_000) == mel.OK
    with pytest.raises(mel.MelError):
        cl.send(3, X, f)
    with pytest.raises(mel.MelError):
        mel.Client("no_such_ring_" + name, 1, 0)
    cl.close()
    ing.destroy()


def test_clients_that_only_finalize_reach_eos(lib):
    """Clients that connect and finalize without sending (an empty simulation) still count
    toward EOS; nothing is returned."""
    n, name = 16, _name()
    ing = mel.Ingest(name, 0, n, slots=4, expected_clients=2)
    for c in (4, 9):
        cl = mel.Client(name, 1, c)
        assert cl.finalize() == mel.OK
        cl.close()
    st, m = ing.next(1000)
    assert st == mel.EOS and m is None
    s = ing.stats()
    assert s["finalized"] == 2 and s["received"] == 0
    ing.destroy()
