"""Multi-process (world_size 2, gloo, CPU) checks of the data-parallel host logic:
round-robin routing of the streamed time steps and the all-reduced
gradient mean of P:171, with per-rank oracle reservoirs fed by their routed share.
Each rank computes its raw SSE gradient on its own Philox batch; the gloo
all-reduce of (grads, SSE, n) must equal the R-rank oracle emulation."""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from mel_inputs import design, heat
from oracle import mlp, reservoir as ores, trainer as otr

WL = design.TINY_EVICT


def _fields():
    X = design.draw_design(WL.sims, seed=1)
    F = {s: heat.simulate(X[s], WL.n, WL.tau) for s in range(WL.sims)}
    return X, F


def _rank_batch(rank, world, X, F, n_puts=150):
    res = ores.Reservoir(WL.capacity, WL.threshold, WL.n_field, seed=1, rank=rank)
    for (s, t) in design.routed_stream(WL.sims, WL.tau, rank, world)[: n_puts // world]:
        res.put(s, t, X[s], F[s][t])
    st, slots = res.sample(WL.batch)
    assert st == ores.OK
    s = np.asarray(slots)
    return mlp.normalise_inputs(res.X[s], res.t[s], WL.tau), ores.stored_to_f64(res.payload[s], 0)


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    X, F = _fields()
    params = mlp.init_params(mlp.layer_dims(WL.n_field, WL.hidden), seed=1)
    xn, tn = _rank_batch(rank, world, X, F)
    S, g = mlp.sse_and_grads(params, xn, tn)
    flat = torch.from_numpy(np.concatenate([x.reshape(-1) for x in mlp.flatten(g)] + [np.array([S, len(xn)])]))
    dist.all_reduce(flat)                         # sum over ranks (the NCCL all-reduce's semantics)
    out[rank] = flat.numpy()
    dist.destroy_process_group()


def test_routing_partitions_the_stream():
    for world in (1, 2, 4, 8):
        parts = [design.routed_stream(WL.sims, WL.tau, r, world) for r in range(world)]
        allp = [p for part in parts for p in part]
        assert sorted(allp) == design.stream_order(WL.sims, WL.tau)          # disjoint cover
        for s in range(WL.sims):                  # balanced per client: floor/ceil(tau/R) steps
            per = [sum(1 for (ss, _) in part if ss == s) for part in parts]
            assert set(per) <= {WL.tau // world, -(-WL.tau // world)}
        if world > 1:   # the first destination depends on the client id
            assert len({design.route(s, 0, world) for s in range(world)}) == world


def test_gloo_allreduce_matches_oracle_data_parallel_step():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    port = 29500 + os.getpid() % 1000
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    X, F = _fields()
    params = mlp.init_params(mlp.layer_dims(WL.n_field, WL.hidden), seed=1)
    tensors = [x.astype(np.float64) for x in mlp.flatten(params)]
    batches = [_rank_batch(r, world, X, F) for r in range(world)]
    loss_o, g_o = otr.global_loss_and_grads(tensors, batches, WL.n_field)
    for r in range(world):
        flat = out[r]
        S, n = flat[-2], flat[-1]
        assert n == world * WL.batch
        assert abs(S / (WL.n_field * n) - loss_o) <= 1e-12 * loss_o
        g = flat[:-2] / (WL.n_field * n)
        np.testing.assert_allclose(g, np.concatenate([x.reshape(-1) for x in g_o]), rtol=1e-10, atol=1e-15)
    assert np.array_equal(out[0], out[1])        # replicas receive identical reduced bytes
