"""Multi-rank GPU parity (run under torchrun, one process per GPU).

Every rank replays the same world-R op-log (time steps routed (sim + t) mod R,
P:212) through its own libmel context; the training step is collective (NCCL
all-reduce of the gradients).  Each process also runs the oracle for ALL
ranks, and checks: its sampled slots bit-exact vs oracle rank r; the global loss
and every weight tensor re-anchored to the oracle's R-rank step; replicas bitwise
identical across ranks (state hash); its reservoir contents bit-exact.

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tests/mp_gpu_parity.py [fp32|bf16]
"""
import hashlib
import os
import sys
from dataclasses import replace

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)


def main():
    import torch
    import torch.distributed as dist

    from harness import FieldTable, compare_reservoir, make_config, rel_norm, tensors_f64
    from mel_inputs import design
    from oracle import mlp, reservoir as ores, trainer as otr
    from paper_2309_16743_b200 import mel

    mode = sys.argv[1] if len(sys.argv) > 1 else "fp32"
    # bf16: in-kernel NVLink exchange (default); bf16-nccl: NCCL reduce-scatter / all-gather
    flags = (mel.FLAG_NCCL_EXCHANGE if mode.endswith("-nccl") else
             mel.FLAG_FP32_EXCHANGE if mode.endswith("-fp32x") else 0)
    # fp32-fifo / fp32-firo: the comparison buffers on every rank
    policy = ores.FIFO if mode.endswith("-fifo") else ores.FIRO if mode.endswith("-firo") else ores.RESERVOIR
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo")
    obj = [mel.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    if mode.startswith("fp32"):
        wl = replace(design.TINY_EVICT, world=world, puts_per_step=10)
        prec = store = 0
        tol_loss, tol_w, max_steps = 1e-5, 1e-5, None
    else:   # bf16, bf16-nccl
        wl = replace(design.MEDIUM, name="medium-bf16-mr", capacity=600, threshold=100, sims=30, world=world,
                     batch=128, puts_per_step=60)
        prec = store = 1
        tol_loss, tol_w, max_steps = 2e-2, 1e-3, 5
    table = FieldTable(wl)
    ctx = mel.Context(make_config(wl, precision=prec, storage=store, flags=flags, policy=policy), rank=rank, world=world,
                      nccl_id=obj[0], device=rank)
    res = [ores.Reservoir(wl.capacity, wl.threshold, wl.n_field, seed=1, rank=r, storage=store, policy=policy)
           for r in range(world)]
    batches = [[] for _ in range(world)]
    steps, worst_l, worst_w = 0, 0.0, 0.0
    for op in design.build_oplog(wl):
        kind = op[0]
        if kind == "PUT":
            _, r, s, t = op
            res[r].put(s, t, table.Xs(s), table.field(s, t))
            if r == rank:
                assert ctx.put(s, t, table.Xs(s), table.field(s, t)) == 0
        elif kind == "CLOSE":
            res[op[1]].close()
            if op[1] == rank:
                ctx.close()
        elif kind == "SAMPLE":
            r = op[1]
            st_o, sl_o = res[r].sample(wl.batch)
            batches[r] = list(sl_o)
            if r == rank:
                st_g, sl_g, n = ctx.sample(want_slots=True)
                assert st_g == st_o and list(sl_g) == list(sl_o), (rank, st_g, st_o)
        elif kind == "STEP":
            n_tot = sum(len(b) for b in batches)
            before = ctx.get_state() if n_tot else None
            st_g, loss_g = ctx.step(want_loss=True)
            if n_tot == 0:
                done = all(r_.over and r_.p == 0 for r_ in res)
                assert st_g == (2 if done else 1), (st_g, done)
                if done:
                    break
                continue
            assert st_g == 0
            rb = []
            for r in range(world):
                if batches[r]:
                    s = np.asarray(batches[r])
                    rb.append((mlp.normalise_inputs(res[r].X[s], res[r].t[s], wl.tau),
                               ores.stored_to_f64(res[r].payload[s], store)))
                else:
                    rb.append(None)
            after = ctx.get_state()
            loss_o, p_o, _, _, _ = otr.one_step_from_state(tensors_f64(before["p"]), tensors_f64(before["m"]),
                                                            tensors_f64(before["v"]), before["k"], before["S"], rb,
                                                            wl.n_field)
            worst_l = max(worst_l, abs(loss_g - loss_o) / loss_o)
            worst_w = max(worst_w, max(rel_norm(a, b) for a, b in zip(tensors_f64(after["p"]), p_o)))
            h = hashlib.sha256(b"".join(x.tobytes() for x in after["p"])).hexdigest()
            hs = [None] * world
            dist.all_gather_object(hs, h)
            assert len(set(hs)) == 1, "replicas diverged"
            batches = [[] for _ in range(world)]
            steps += 1
            if max_steps and steps >= max_steps:
                break
    compare_reservoir(ctx, res[rank], store)
    assert steps > 3 and worst_l <= tol_loss and worst_w <= tol_w, (steps, worst_l, worst_w)
    print("rank %d/%d %s: %d steps, loss err %.2e, weight err %.2e, replicas identical" %
          (rank, world, mode, steps, worst_l, worst_w), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
