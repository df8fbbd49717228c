"""Seeded synthetic client payloads for the ingest channel: what a
simulation client hands to `send` before the fp64 -> fp32 conversion.
Values are fp64 kelvin in the workload's [100, 500) range with all 52 mantissa bits
populated, so the wire rounding is exercised on every element."""
from __future__ import annotations

import numpy as np

from .design import T_HI, T_LO


def client_X(client: int, seed: int = 0) -> np.ndarray:
    rng = np.random.default_rng([int(seed), 7, int(client)])
    return (T_LO + (T_HI - T_LO) * rng.random(5)).astype(np.float32)


def client_field(client: int, t: int, n_field: int, seed: int = 0) -> np.ndarray:
    rng = np.random.default_rng([int(seed), 11, int(client), int(t)])
    return T_LO + (T_HI - T_LO) * rng.random(n_field)
