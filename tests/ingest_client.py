"""A simulation client process for the ingest tests and tools/ingest_bench.py:
init_communication, send of t in [t0, t1) (fp64 payloads from mel_inputs.clients),
optionally finalize_communication."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from mel_inputs import clients  # noqa: E402
from paper_2309_16743_b200 import mel  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("name")
ap.add_argument("world", type=int)
ap.add_argument("client", type=int)
ap.add_argument("t0", type=int)
ap.add_argument("t1", type=int)
ap.add_argument("--n-field", type=int, required=True)
ap.add_argument("--finalize", action="store_true")
ap.add_argument("--seed", type=int, default=0)
ap.add_argument("--cycle", type=int, default=0, help="reuse this many pre-generated payloads (bench)")
a = ap.parse_args()

cl = mel.Client(a.name, a.world, a.client)
X = clients.client_X(a.client, a.seed)
pre = [clients.client_field(a.client, t, a.n_field, a.seed) for t in range(a.cycle)] if a.cycle else None
for t in range(a.t0, a.t1):
    f = pre[t % a.cycle] if pre else clients.client_field(a.client, t, a.n_field, a.seed)
    if cl.send(t, X, f, timeout_us=60_000_000) != mel.OK:
        sys.exit(2)
if a.finalize:
    cl.finalize(timeout_us=60_000_000)
cl.close()
