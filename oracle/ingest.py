"""ORACLE (test infrastructure only -- never imported by the product path).

The ingest step before the training buffer, as the paper states it:

  * conversion on the client, "typically from 64 to 32 bits":
    fp32 = round-to-nearest-even of the fp64 value (numpy's cast is that rounding);
  * round-robin distribution over the server ranks, first destination from the client
    id, reading R10: rank(c, t) = (c + t) mod R;
  * the per-client log of received messages, "in case of client restart, already
    received messages are discarded", reading R23: key (client, t); a rank keeps
    the first copy of each key, in arrival order.

`server_accept` is the whole server-side semantics of one rank given the sequence of
messages that reached it; `rank_streams` applies the routing to per-client send logs.
Pinned in tests/test_oracle_ingest.py (round-robin balance and first destination,
brute force on tiny logs, fp32 rounding special cases).
"""
from __future__ import annotations

import numpy as np


def route(client: int, t: int, world: int) -> int:
    """P:212 + reading R10."""
    return (client + t) % world


def to_wire(field_f64) -> np.ndarray:
    """the client converts its fp64 field to fp32 (RNE)."""
    return np.asarray(field_f64, dtype=np.float64).astype(np.float32)


def rank_streams(sends, world: int) -> list[list[tuple[int, int]]]:
    """sends: (client, t) in send order (any interleaving of clients, restarts included).
    Returns, per rank, the (client, t) keys that reach it, in that order."""
    out = [[] for _ in range(world)]
    for c, t in sends:
        out[route(c, t, world)].append((c, t))
    return out


def server_accept(arrivals) -> list[tuple[int, int]]:
    """P:183 + reading R23: the first copy of every (client, t), in arrival order."""
    log = set()
    kept = []
    for key in arrivals:
        if key in log:
            continue
        log.add(key)
        kept.append(key)
    return kept
