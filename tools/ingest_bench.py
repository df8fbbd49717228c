"""Sustained ingest throughput of the f2 path: P client processes
(tests/ingest_client.py: fp64 payload -> fp32 conversion in the client) stream
paper-shaped time steps (N = 10^6) into one rank's shared-memory ring; the server
drains it with reservoir_ingest (DMA from the page-locked segment into the staging ring,
commit into the bf16 reservoir).  Two phases:
  ingest-only : the server loop is reservoir_ingest + a commit point (sample) per call;
  with-train  : the same plus one surrogate_step per call (the paper's concurrent
                reception and training).
Prints one JSON line per phase: messages/s, wire GB/s (fp32 payload), clients, slots.
"""
import argparse
import json
import os
import subprocess
import sys
import time
import uuid

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2309_16743_b200 import mel  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--clients", type=int, default=max(1, min(16, (os.cpu_count() or 4) - 4)))
ap.add_argument("--steps", type=int, default=200, help="time steps per client")
ap.add_argument("--n-field", type=int, default=1_000_000)
ap.add_argument("--slots", type=int, default=32)
ap.add_argument("--batch", type=int, default=1024)
ap.add_argument("--max-msgs", type=int, default=16)
a = ap.parse_args()


def phase(train: bool):
    name = "b" + uuid.uuid4().hex[:10]
    ing = mel.Ingest(name, 0, a.n_field, a.slots, expected_clients=a.clients)
    cfg = mel.Config(n_field=a.n_field, batch=a.batch, capacity=6000, threshold=1000, precision=mel.BF16,
                     storage=mel.STORE_BF16, staging_entries=max(64, a.max_msgs + 8), steps_per_sim=100)
    ctx = mel.Context(cfg)
    cmd = [sys.executable, os.path.join(ROOT, "tests", "ingest_client.py"), name, "1"]
    procs = [subprocess.Popen(cmd + [str(c), "0", str(a.steps), "--n-field", str(a.n_field), "--finalize",
                                     "--cycle", "2"]) for c in range(a.clients)]
    n, steps, t0 = 0, 0, None
    while True:
        st, k = ctx.ingest(ing, max_msgs=a.max_msgs, timeout_us=60_000_000)
        if st == mel.EOS:
            break
        if t0 is None and k:
            t0 = time.perf_counter()       # the clock starts at the first message
        n += k
        r, _, _ = ctx.sample()
        if train and r == mel.OK:
            ctx.step(want_loss=False)
            steps += 1
    ctx.sync()
    dt = time.perf_counter() - t0
    ok = all(p.wait(120) == 0 for p in procs)
    s = ing.stats()
    ing.destroy()
    return {"phase": "with-train" if train else "ingest-only", "clients": a.clients, "slots": a.slots,
            "n_field": a.n_field, "messages": n, "seconds": round(dt, 3), "msgs_per_s": round(n / dt, 1),
            "wire_GB_per_s": round(n * 4 * a.n_field / dt / 1e9, 2), "train_steps": steps,
            "duplicates": s["duplicates"], "clients_ok": ok}


for train in (False, True):
    print(json.dumps(phase(train)), flush=True)
