"""GPU parity of the ingest path: client processes -> shared-memory
ring -> reservoir_ingest (DMA from the page-locked segment) -> the buffer, bit-exact
against the oracle reservoir fed the same first-copy messages in the same order
(oracle/ingest.py for the wire conversion and the log)."""
import os
import subprocess
import sys
import uuid

import numpy as np
import pytest

from harness import compare_reservoir
from mel_inputs import clients
from oracle import ingest as oi, reservoir as ores
from paper_2309_16743_b200 import mel

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLIENT = os.path.join(ROOT, "tests", "ingest_client.py")


def _spawn(name, world, client, t0, t1, n, finalize=True):
    cmd = [sys.executable, CLIENT, name, str(world), str(client), str(t0), str(t1), "--n-field", str(n)]
    return subprocess.Popen(cmd + (["--finalize"] if finalize else []))


@pytest.mark.parametrize("storage", [mel.STORE_F32, mel.STORE_BF16])
def test_single_client_ingest_with_eviction_bit_exact(storage):
    """One client restarting once (t = 0..9, then 0..149): evictions, the watermark,
    a 4-entry staging ring that fills inside reservoir_ingest, duplicates dropped."""
    n, C, theta, B, name = 100, 48, 8, 8, "g" + uuid.uuid4().hex[:10]
    ing = mel.Ingest(name, 0, n, slots=16, expected_clients=1)
    ctx = mel.Context(mel.Config(n_field=n, hidden=(32,), capacity=C, threshold=theta, batch=B, steps_per_sim=150,
                                 storage=storage, seed=3, staging_entries=4))
    res = ores.Reservoir(C, theta, n, seed=3, storage=storage)
    assert _spawn(name, 1, 9, 0, 10, n, finalize=False).wait(120) == 0
    p = _spawn(name, 1, 9, 0, 150, n)
    X = clients.client_X(9)
    t_next, calls = 0, 0
    while True:
        st, k = ctx.ingest(ing, max_msgs=6, timeout_us=20_000_000)
        if st == mel.EOS:
            break
        for t in range(t_next, t_next + k):          # one client: first copies arrive in t order
            res.put(9, t, X, oi.to_wire(clients.client_field(9, t, n)))
        t_next += k
        calls += 1
        a, sa, _ = ctx.sample(want_slots=True)
        b, sb = res.sample(B)
        assert a == b and list(sa) == list(sb)
    assert p.wait(120) == 0
    assert t_next == 150 and calls >= 150 // 6
    s = ing.stats()
    assert s["received"] == 150 and s["duplicates"] == 10
    ctx.close(); res.close()
    compare_reservoir(ctx, res, storage=storage)
    ing.destroy()


def test_many_clients_ingest_arrival_order_bit_exact():
    """Six concurrent client processes: the buffer (no eviction) holds the first copies
    in the ring's arrival order, so slot j = j-th arrival; the oracle fed that order
    reproduces every slot bit for bit, and the keys are exactly the routed sends."""
    n, nc, tau, name = 256, 6, 30, "g" + uuid.uuid4().hex[:10]
    C = nc * tau + 20
    ing = mel.Ingest(name, 0, n, slots=8, expected_clients=nc)
    ctx = mel.Context(mel.Config(n_field=n, hidden=(32,), capacity=C, threshold=10, batch=4, steps_per_sim=tau,
                                 seed=5, staging_entries=32))
    procs = [_spawn(name, 1, c, 0, tau, n) for c in range(nc)]
    ks = []
    while True:
        st, k = ctx.ingest(ing, max_msgs=32, timeout_us=20_000_000)
        if st == mel.EOS:
            break
        ks.append(k)
        ctx.sample()                                  # commit point
    total = sum(ks)
    assert all(p.wait(120) == 0 for p in procs)
    assert total == nc * tau
    ctx.close()
    d = ctx.dump(payload=False)
    order = list(zip(d["sim"][:total].tolist(), d["t"][:total].tolist()))
    assert sorted(order) == sorted(oi.server_accept(oi.rank_streams([(c, t) for c in range(nc)
                                                                      for t in range(tau)], 1)[0]))
    # independent of the slot dump's own order: every client sends t = 0, 1, ... in sequence
    # and takes its ring tickets in that order, so the ring must hand each client's messages
    # over in send order (a permutation inside the ring breaks this)
    for c in range(nc):
        assert [t for (s, t) in order if s == c] == list(range(tau)), c
    res = ores.Reservoir(C, 10, n, seed=5)
    i = 0
    for k in ks:                                      # the same puts between the same commit points
        for c, t in order[i:i + k]:
            res.put(c, t, clients.client_X(c), oi.to_wire(clients.client_field(c, t, n)))
        i += k
        res.sample(4)
    res.close()
    compare_reservoir(ctx, res)
    ing.destroy()
