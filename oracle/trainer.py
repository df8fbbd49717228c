"""ORACLE (test infrastructure only -- never imported by the product path).

Data-parallel online training as the server of the paper runs it ("All MPI
processes run an identical copy of the NN ... the locally computed vector of
weight updates is all-reduced", P:173 training thread, P:177 one buffer per
server process, P:212 round-robin routing), emulated with R logical ranks.

Readings (R10-R12):
  * per step rank r contributes n_r samples (B during reception, <= B while
    draining, 0 after EAGAIN);
  * global loss      L = sum_r SSE_r / (N * sum_r n_r);
  * global gradient  g = (rank-ordered sum of raw dSSE_r) / (N * sum_r n_r),
    which equals the mean of per-rank means when every n_r = B (DDP);
  * Adam + LR schedule on the global gradient (oracle.mlp), S counts global
    samples (P:414 n_s = n_b * b * n_GPU);
  * EOS when every rank is over and empty; a step with sum n_r = 0 otherwise is
    a no-op (SKIP).
"""
from __future__ import annotations

import numpy as np

from . import mlp
from .reservoir import EAGAIN, OK, Reservoir, stored_to_f64

SKIP, EOS = 1, 2


class Trainer:
    def __init__(self, n_field: int, hidden, tau: int, capacity: int, threshold: int,
                 batch: int, world: int = 1, seed: int = 1, storage: int = 0, params=None):
        self.N, self.tau, self.B, self.R = n_field, tau, batch, world
        self.dims = mlp.layer_dims(n_field, hidden)
        self.res = [Reservoir(capacity, threshold, n_field, seed=seed, rank=r, storage=storage)
                    for r in range(world)]
        p32 = params if params is not None else mlp.init_params(self.dims, seed)
        self.tensors = [np.asarray(x, np.float32).astype(np.float64) for x in mlp.flatten(p32)]
        self.adam = mlp.Adam(self.tensors)
        self.S = 0
        self.batches = [[] for _ in range(world)]
        self.losses: list[float] = []
        self.lrs: list[float] = []

    # -- buffer side ----------------------------------------------------------------
    def put(self, rank, sim, t, X, field):
        return self.res[rank].put(sim, t, X, field)

    def close(self, rank):
        return self.res[rank].close()

    def sample(self, rank):
        st, slots = self.res[rank].sample(self.B)
        self.batches[rank] = slots if st == OK else []
        return st, slots

    def batch_arrays(self, rank, slots):
        r = self.res[rank]
        s = np.asarray(slots, dtype=np.int64)
        xn = mlp.normalise_inputs(r.X[s], r.t[s], self.tau)
        tn = stored_to_f64(r.payload[s], r.storage)
        return xn, tn

    # -- training side --------------------------------------------------------------
    def step(self):
        n = [len(b) for b in self.batches]
        n_tot = sum(n)
        if n_tot == 0:
            done = all(r.over and r.p == 0 for r in self.res)
            self.batches = [[] for _ in range(self.R)]
            return (EOS if done else SKIP), None
        loss, grads = global_loss_and_grads(self.tensors, [self.batch_arrays(r, b) if b else None
                                                           for r, b in enumerate(self.batches)], self.N)
        lr = mlp.lr_schedule(self.S)
        self.tensors = self.adam.step(self.tensors, grads, lr)
        self.S += n_tot
        self.losses.append(loss)
        self.lrs.append(lr)
        self.batches = [[] for _ in range(self.R)]
        return OK, loss


def global_loss_and_grads(tensors, rank_batches, n_field):
    """rank_batches: list over ranks of (xn, tn) or None.  Rank-ordered sums."""
    params = mlp.unflatten(tensors)
    S_tot, g_tot, n_tot = 0.0, None, 0
    for rb in rank_batches:
        if rb is None:
            continue
        xn, tn = rb
        S, g = mlp.sse_and_grads(params, xn, tn)
        g = mlp.flatten(g)
        S_tot += S
        g_tot = g if g_tot is None else [a + b for a, b in zip(g_tot, g)]
        n_tot += xn.shape[0]
    denom = float(n_field) * n_tot
    return S_tot / denom, [x / denom for x in g_tot]


def one_step_from_state(tensors, m, v, k_before: int, S_before: int, rank_batches, n_field):
    """Re-anchored single step: run step k = k_before + 1 in
    fp64 from an externally supplied state (e.g. the GPU's fp32 state promoted).
    Returns (loss, new_tensors, new_m, new_v, lr)."""
    loss, grads = global_loss_and_grads(tensors, rank_batches, n_field)
    lr = mlp.lr_schedule(S_before)
    out_p, out_m, out_v = [], [], []
    for p, g, mm, vv in zip(tensors, grads, m, v):
        p2, m2, v2 = mlp.adam_update(p, g, mm, vv, k_before + 1, lr)
        out_p.append(p2); out_m.append(m2); out_v.append(v2)
    return loss, out_p, out_m, out_v, lr


def replay(trainer: Trainer, ops, field_of, X_of, on_step=None):
    """Run an op-log (mel_inputs.design.build_oplog) through the oracle.
    field_of(sim, t) -> fp32 field; X_of(sim) -> fp32 X[5].  Returns the trace."""
    trace = dict(sample=[], step=[])
    for op in ops:
        kind = op[0]
        if kind == "PUT":
            _, r, s, t = op
            trainer.put(r, s, t, X_of(s), field_of(s, t))
        elif kind == "SAMPLE":
            st, slots = trainer.sample(op[1])
            trace["sample"].append((op[1], st, list(slots)))
        elif kind == "CLOSE":
            trainer.close(op[1])
        elif kind == "STEP":
            st, loss = trainer.step()
            trace["step"].append((st, loss))
            if on_step is not None:
                on_step(trainer, st, loss)
            if st == EOS:
                break
    return trace
