"""Multi-rank ingest (run under torchrun, one process per GPU): client processes stream
their time steps round robin over every rank's shared-memory ring (reading R10),
each rank drains its ring with reservoir_ingest and trains collectively.
Checks per rank: the first copies that reached it are exactly its routed keys, its
buffer is bit-exact against the oracle reservoir fed the observed arrival order with the
same commit points, and the replicas stay bitwise identical (state hash every 8 steps).

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tests/mp_gpu_ingest.py
"""
import hashlib
import os
import subprocess
import sys
import uuid

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)


def main():
    import torch
    import torch.distributed as dist

    from harness import compare_reservoir
    from mel_inputs import clients
    from oracle import ingest as oi, reservoir as ores
    from paper_2309_16743_b200 import mel

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo")
    obj = [(mel.nccl_unique_id(), "m" + uuid.uuid4().hex[:10]) if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    nccl_id, name = obj[0]
    n, nc, tau, B = 1024, 6, 20, 16
    C = nc * tau                                       # no eviction: slot j = j-th arrival
    ing = mel.Ingest(name, rank, n, slots=8, expected_clients=nc)
    cfg = mel.Config(n_field=n, hidden=(64, 64), capacity=C, threshold=8, batch=B, steps_per_sim=tau, seed=4,
                     staging_entries=32)
    ctx = mel.Context(cfg, rank=rank, world=world, nccl_id=nccl_id, device=rank)
    dist.barrier()
    procs = []
    if rank == 0:
        for c in range(nc):
            procs.append(subprocess.Popen([sys.executable, os.path.join(HERE, "ingest_client.py"), name, str(world),
                                           str(c), "0", str(tau), "--n-field", str(n), "--finalize"]))
    ks, steps, eos = [], 0, False
    while True:
        st, k = (mel.EOS, 0) if eos else ctx.ingest(ing, max_msgs=8, timeout_us=2000)
        eos = eos or st == mel.EOS
        ks.append(k)
        ctx.sample()                                    # commit point (and a batch once p > theta)
        r, _ = ctx.step(want_loss=False)                # collective: every rank steps every round
        steps += r == mel.OK
        if steps % 8 == 0:
            h = hashlib.sha256(b"".join(x.tobytes() for x in ctx.get_state()["p"])).hexdigest()
            hs = [None] * world
            dist.all_gather_object(hs, h)
            assert len(set(hs)) == 1, "replicas diverged"
        done = torch.tensor([1 if eos else 0])
        dist.all_reduce(done)
        if int(done) == world:
            break
    assert all(p.wait(120) == 0 for p in procs)
    ctx.sync()
    total = sum(ks)
    sends = [(c, t) for c in range(nc) for t in range(tau)]
    d = ctx.dump(payload=False)
    order = list(zip(d["sim"][:total].tolist(), d["t"][:total].tolist()))
    assert sorted(order) == sorted(oi.rank_streams(sends, world)[rank]), "rank %d got other keys" % rank
    res = ores.Reservoir(C, 8, n, seed=4, rank=rank)
    i = 0
    for k in ks:
        for c, t in order[i:i + k]:
            res.put(c, t, clients.client_X(c), oi.to_wire(clients.client_field(c, t, n)))
        i += k
        res.sample(B)
    compare_reservoir(ctx, res)
    hs = [None] * world
    dist.all_gather_object(hs, hashlib.sha256(b"".join(x.tobytes() for x in ctx.get_state()["p"])).hexdigest())
    assert len(set(hs)) == 1
    print("rank %d/%d ingest: %d messages, %d steps, replicas identical" % (rank, world, total, steps), flush=True)
    ing.destroy()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
