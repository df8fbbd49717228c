"""ORACLE -- test infrastructure only.

A plain, slow, obviously-correct CPU (numpy fp64) implementation of the hot path
of arXiv 2309.16743 (Meyer et al., "High Throughput Training of Deep Surrogates
from Large Ensemble Runs"), written from PAPER.md: the Reservoir (Algorithm 1),
Philox-driven sampling, the MLP surrogate's forward/backward, Adam with the LR
schedule, and the data-parallel gradient mean; plus the §8(f) rows' semantics:
the ingest routing / wire conversion / restart log (`ingest`) and the offline
baseline's epoch order (`dataset`).

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
`--impl reference` legs may import it.  The product package
(`paper_2309_16743_b200`) never imports, links or executes anything here, and
this package never imports the product.  Both consume the seeded input
generators in `mel_inputs/`, which hold none of the method's arithmetic.

Parity status per function: see DESIGN.md "Oracle pins".  Every function is
pinned by a -m "not gpu" test except the multi-step training trajectory
("parity unpinned" beyond the per-step pins -- the paper prints no trajectory).
"""
from . import dataset, ingest, mlp, philox, reservoir, trainer  # noqa: F401
