"""Test harness: replay one op-log (mel_inputs.design) through the CUDA path (via
the C ABI binding) and through the oracle, side by side.  Only tests import this
module; it never feeds a value from the CUDA path into the oracle except the
re-anchored state (the oracle runs step k in fp64 from the
GPU's exact fp32 state after step k-1), which is an INPUT to the oracle step,
never an expected value."""
from __future__ import annotations

import numpy as np

from mel_inputs import design, heat
from oracle import mlp, reservoir as ores, trainer as otr


class FieldTable:
    """Exact heat-equation fields for a workload (direct solves for small grids,
    the linear basis for larger ones)."""

    def __init__(self, wl: design.Workload, seed: int = 1):
        self.wl = wl
        self.X = design.draw_design(wl.sims, seed=seed)
        self.phi = None
        self.cache = {}
        if wl.n <= 16:
            for s in range(wl.sims):
                self.cache[s] = heat.simulate(self.X[s], wl.n, wl.tau)
        else:
            self.phi = heat.basis(wl.n, wl.tau)

    def field(self, s, t):
        if self.phi is None:
            return self.cache[s][t]
        return heat.fields_from_basis(self.phi, self.X[s], t)

    def Xs(self, s):
        return self.X[s]


def make_config(wl: design.Workload, precision=0, storage=0, seed=1, staging=None, flags=0, batch=None, policy=0):
    # the op-log holds puts_per_step puts pending between commit points
    staging = staging or wl.puts_per_step + 8
    from paper_2309_16743_b200 import mel
    return mel.Config(n_field=wl.n_field, hidden=wl.hidden, capacity=wl.capacity, threshold=wl.threshold,
                      batch=batch or wl.batch, steps_per_sim=wl.tau, precision=precision, storage=storage,
                      seed=seed, staging_entries=staging, flags=flags, policy=policy)


def tensors_f64(st):
    return [np.asarray(x, np.float32).astype(np.float64) for x in st]


def rel_norm(a, b):
    a = np.asarray(a, np.float64).reshape(-1)
    b = np.asarray(b, np.float64).reshape(-1)
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (nb if nb > 0 else 1.0))


def tile_errors(a, b, rows_per_tile=128):
    """W_L (rows = output neurons) compared per 128-row tile (one K1 tile / one exchange
    unit): the worst tile's relative norm error and the element-wise max abs error."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    a2, b2 = a.reshape(a.shape[0], -1), b.reshape(b.shape[0], -1)
    worst = 0.0
    for r0 in range(0, a2.shape[0], rows_per_tile):
        worst = max(worst, rel_norm(a2[r0:r0 + rows_per_tile], b2[r0:r0 + rows_per_tile]))
    return worst, float(np.max(np.abs(a2 - b2))) if a2.size else 0.0


def replay_parity(ctx, wl, table, ops, storage=0, seed=1, reanchor=True, max_train_steps=None,
                  on_step=None, check_every_sample=True, policy=0):
    """Drive ctx (world 1) and an oracle reservoir with the same op-log.  Returns a
    report dict; asserts bit-exact sampling on the way."""
    res = ores.Reservoir(wl.capacity, wl.threshold, wl.n_field, seed=seed, rank=0, storage=storage, policy=policy)
    report = dict(loss_err=[], w_err=[], tile_err=[], max_abs=[], steps=0, samples=0, eagain=0)
    last_slots = []
    S_host = 0
    k_host = 0
    for op in ops:
        kind = op[0]
        if kind == "PUT":
            _, r, s, t = op
            f = table.field(s, t)
            assert ctx.put(s, t, table.Xs(s), f) == 0
            res.put(s, t, table.Xs(s), f)
        elif kind == "CLOSE":
            ctx.close()
            res.close()
        elif kind == "SAMPLE":
            st_o, slots_o = res.sample(wl.batch)
            st_g, slots_g, n_g = ctx.sample(want_slots=True)
            assert st_g == st_o, (st_g, st_o)
            assert n_g == len(slots_o), (n_g, len(slots_o))
            assert np.array_equal(slots_g.astype(np.int64), np.asarray(slots_o, dtype=np.int64)), "slot mismatch"
            last_slots = list(slots_o)
            if st_o == ores.EAGAIN:
                report["eagain"] += 1
        elif kind == "STEP":
            if not last_slots:
                st_g, _ = ctx.step(want_loss=True)
                if res.over and res.p == 0:
                    assert st_g == 2, st_g      # EOS
                    break
                assert st_g == 1, st_g          # nothing to train on
                continue
            before = ctx.get_state() if reanchor else None
            st_g, loss_g = ctx.step(want_loss=True)
            assert st_g == 0
            s = np.asarray(last_slots)
            xn = mlp.normalise_inputs(res.X[s], res.t[s], wl.tau)
            tn = ores.stored_to_f64(res.payload[s], storage)
            if reanchor:
                after = ctx.get_state()
                assert after["k"] == before["k"] + 1 and after["S"] == before["S"] + len(s)
                loss_o, p_o, _, _, _ = otr.one_step_from_state(
                    tensors_f64(before["p"]), tensors_f64(before["m"]), tensors_f64(before["v"]),
                    before["k"], before["S"], [(xn, tn)], wl.n_field)
                report["loss_err"].append(abs(loss_g - loss_o) / loss_o)
                got = tensors_f64(after["p"])
                report["w_err"].append(max(rel_norm(a, b) for a, b in zip(got, p_o)))
                te, ma = tile_errors(got[-2], p_o[-2])          # W_L per 128-row tile
                report["tile_err"].append(te)
                report["max_abs"].append(ma)
            if on_step is not None:
                on_step(ctx, res, loss_g, s)
            report["steps"] += 1
            report["samples"] += len(s)
            last_slots = []
            if max_train_steps is not None and report["steps"] >= max_train_steps:
                break
    report["oracle_res"] = res
    return report


def compare_reservoir(ctx, res, storage=0):
    """Bit-exact comparison of every slot's metadata, seen counter, put_seq and
    stored payload, plus the counters."""
    d = ctx.dump(payload=True)
    C = res.C
    occupied = res.sim >= 0
    assert np.array_equal(d["sim"][occupied].astype(np.int64), res.sim[occupied])
    assert np.array_equal(d["t"][occupied].astype(np.int64), res.t[occupied])
    assert np.array_equal(d["X"][occupied].view(np.uint32), res.X[occupied].view(np.uint32))
    assert np.array_equal(d["seen"][occupied].astype(np.int64), res.seen[occupied])
    assert np.array_equal(d["put_seq"][occupied].astype(np.int64), res.put_seq[occupied])
    if storage == 0:
        assert np.array_equal(d["payload"][occupied].view(np.uint32), res.payload[occupied].view(np.uint32))
    else:
        assert np.array_equal(d["payload"][occupied], res.payload[occupied])
    s = ctx.stats()
    o = res.stats()
    for k in ("population", "unseen", "seen", "puts", "committed", "draws", "evictions", "pending"):
        assert s[k] == o[k], (k, s[k], o[k])
    assert np.array_equal(s["hist"], o["hist"])
