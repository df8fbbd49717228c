"""ORACLE (test infrastructure only -- never imported by the product path).

The offline baseline's data order (§4.4 "Online versus multi-epoch Offline",
P:425-469): the same trainer, fed by epochs over a fixed dataset stored beforehand.
The paper does not state its shuffle; reading R24 fixes it as the
Fisher-Yates / Durstenfeld shuffle of the identity driven by the library's Philox stream
(reading Q8), tag TAG_EPOCH, counter i, c2 = epoch:

    perm = [0, 1, ..., n-1]
    for i = n-1 down to 1:
        j = bounded(r64(seed, TAG_EPOCH, i, epoch), i + 1)
        swap(perm[i], perm[j])

and batch b of an epoch = perm[b*B : (b+1)*B] for b < n // B (the last partial batch is
dropped).  Pinned in tests/test_oracle_dataset.py (a permutation; every draw sequence
gives a distinct permutation -- Fisher-Yates is a bijection from draws to orders --
checked exhaustively for n <= 5; uniform frequencies over many seeds for n = 3).
"""
from __future__ import annotations

import numpy as np

from . import philox


def epoch_order(n: int, seed: int, epoch: int, chooser=None) -> np.ndarray:
    """chooser(i) -> j in [0, i] replaces the Philox draw (tests inject one)."""
    if chooser is None:
        i = np.arange(n, dtype=np.uint64)
        r = philox.r64(seed, philox.TAG_EPOCH, i, epoch)          # r[i] = the draw at step i

        def chooser(k):
            return int(philox.bounded(r[k], k + 1))
    perm = list(range(n))
    for i in range(n - 1, 0, -1):
        j = chooser(i)
        perm[i], perm[j] = perm[j], perm[i]
    return np.asarray(perm, dtype=np.int64)


def batches(n: int, B: int, seed: int, epoch: int) -> list[np.ndarray]:
    perm = epoch_order(n, seed, epoch)
    return [perm[b * B:(b + 1) * B] for b in range(n // B)]
