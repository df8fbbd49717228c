"""Seeded synthetic input generators (heat-equation clients, experimental design,
op-log schedules).  Shared by `oracle/` tests, the GPU parity tests and
`bench.py`; contains none of the method's arithmetic (reservoir, sampler, MLP,
optimiser), so it couples neither side to the other."""
from . import design, heat  # noqa: F401
