"""Seeded synthetic-input generator: experimental design, routing and op-log
schedules.  Shared by the oracle tests, the GPU parity tests and the bench; it
holds none of the method's arithmetic.

Paper anchors:
  * P:175  Monte Carlo experimental design (the aggregator "controls the
           experimental design").  X ~ U[100, 500)^5 K.
  * P:212  "distributes the produced time steps across all GPUs in a Round-Robin
           fashion. The destination of the first time step is chosen according
           to the client id" -> rank(sim, t) = (sim + t) mod R (reading Q10).
  * P:202  intra-simulation order: a client emits t = 0, 1, ... in order.
  * P:360  validation: 10 held-out simulations.

The op-log is the deterministic interleaving (reading Q4) both the oracle and the
CUDA path consume: ("PUT", rank, sim, t), ("SAMPLE", rank), ("STEP",),
("CLOSE", rank).  Payloads are looked up by (sim, t) in a field table.
"""
from __future__ import annotations

from dataclasses import dataclass, field as dc_field

import numpy as np

T_LO, T_HI = 100.0, 500.0


def draw_design(n_sims: int, seed: int, validation: bool = False) -> np.ndarray:
    """Monte Carlo design: (n_sims, 5) fp32 kelvin in [100, 500)."""
    rng = np.random.default_rng([int(seed), 1 if validation else 0])
    return (T_LO + (T_HI - T_LO) * rng.random((n_sims, 5))).astype(np.float32)


def route(sim: int, t: int, world: int) -> int:
    """Round-robin routing of a client's time steps (reading Q10)."""
    return (sim + t) % world


@dataclass
class Workload:
    name: str
    n: int                 # grid nodes per axis (field N = n*n)
    tau: int               # time steps per simulation
    sims: int
    hidden: tuple
    capacity: int
    threshold: int
    batch: int
    puts_per_step: int
    world: int = 1
    extra: dict = dc_field(default_factory=dict)

    @property
    def n_field(self) -> int:
        return self.n * self.n


# BASELINE.json configs; theta follows the paper's 1000/6000
# ratio where BASELINE is silent.
TINY = Workload("tiny", 10, 10, 20, (32,), 200, 33, 8, 5)
TINY_EVICT = Workload("tiny-evict", 10, 10, 20, (32,), 48, 8, 8, 5)
MEDIUM = Workload("medium", 100, 100, 1000, (256, 256), 50000, 8333, 256, 100)
PAPER = Workload("paper-shaped", 1000, 100, 10000, (256, 256), 6000, 1000, 1024, 4)


def stream_order(n_sims: int, tau: int) -> list[tuple[int, int]]:
    """Arrival order of (sim, t): simulations in order, t ascending."""
    return [(s, t) for s in range(n_sims) for t in range(tau)]


def build_oplog(wl: Workload, n_steps_after_close: int | None = None,
                max_steps: int | None = None) -> list[tuple]:
    """Deterministic schedule: k PUTs (routed) per STEP; every STEP is preceded by
    one SAMPLE per rank.  After the last put every rank CLOSEs, then SAMPLE+STEP
    repeat until every rank is drained (the consumer detects EOS; we emit a
    generous number of drain steps and the replayer stops at global EOS)."""
    order = stream_order(wl.sims, wl.tau)
    ops: list[tuple] = []
    k = wl.puts_per_step
    steps = 0
    for i in range(0, len(order), k):
        for (s, t) in order[i:i + k]:
            ops.append(("PUT", route(s, t, wl.world), s, t))
        for r in range(wl.world):
            ops.append(("SAMPLE", r))
        ops.append(("STEP",))
        steps += 1
        if max_steps is not None and steps >= max_steps:
            return ops
    for r in range(wl.world):
        ops.append(("CLOSE", r))
    if n_steps_after_close is None:
        n_steps_after_close = wl.capacity // max(1, wl.batch) + 4
    for _ in range(n_steps_after_close):
        for r in range(wl.world):
            ops.append(("SAMPLE", r))
        ops.append(("STEP",))
    return ops


def routed_stream(n_sims: int, tau: int, rank: int, world: int) -> list[tuple[int, int]]:
    """The (sim, t) time steps one server rank receives, in arrival order: the
    global stream (sims in order, t ascending) filtered by the round-robin route."""
    return [(s, t) for s in range(n_sims) for t in range(tau) if route(s, t, world) == rank]
