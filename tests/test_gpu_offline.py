"""GPU parity of the offline baseline: a file dataset ->
epoch-ordered loader threads -> FIFO batches -> the same trainer.  Each epoch's batches
must be exactly oracle/dataset.py's order (checked through the FIFO hand-out), and the
free-running fp32 losses/weights must follow the fp64 oracle chain from the same
initial state within the fp32 bar (1e-5)."""
import numpy as np
import pytest

from harness import rel_norm, tensors_f64
from mel_inputs import clients
from oracle import dataset as od, mlp, reservoir as ores, trainer as otr
from paper_2309_16743_b200 import mel

pytestmark = pytest.mark.gpu


def _records(n_sims, tau, n):
    out = []
    for s in range(n_sims):
        X = clients.client_X(s)
        for t in range(tau):
            out.append((s, t, X, clients.client_field(s, t, n).astype(np.float32)))
    return out


@pytest.mark.parametrize("precision", [mel.FP32, mel.BF16])
def test_offline_epochs_follow_the_oracle(tmp_path, precision):
    # fp32: 60 records = 3 batches of 16 + a dropped tail of 12; bf16 (tcgen05 output
    # layer): 200 records = 3 batches of 64 + a dropped tail of 8
    if precision == mel.FP32:
        n, n_sims, hidden, B = 100, 6, (32, 32), 16
    else:
        n, n_sims, hidden, B = 1024, 20, (256, 256), 64
    tau, seed = 10, 11
    recs = _records(n_sims, tau, n)
    path = str(tmp_path / "ds.bin")
    mel.write_dataset(path, n, recs)
    ds = mel.Dataset(path, threads=4)
    cfg = mel.Config(n_field=n, hidden=hidden, capacity=2 * B, threshold=0, batch=B, steps_per_sim=tau,
                     precision=precision, storage=mel.STORE_BF16 if precision == mel.BF16 else mel.STORE_F32,
                     seed=seed, staging_entries=2 * B, policy=mel.FIFO)
    ctx = mel.Context(cfg)
    st = ctx.get_state()
    p, m, v = tensors_f64(st["p"]), tensors_f64(st["m"]), tensors_f64(st["v"])
    k, S = st["k"], st["S"]
    losses_o = []
    res = ores.Reservoir(2 * B, 0, n, seed=seed, storage=cfg.storage, policy=ores.FIFO)
    for epoch in range(2):
        steps, losses_g = ctx.train_offline(ds, seed=seed, epoch=epoch)
        assert steps == len(recs) // B
        for b in od.batches(len(recs), B, seed, epoch):
            for i in b:
                s_, t_, X_, f_ = recs[i]
                res.put(s_, t_, X_, f_)
            stt, slots = res.sample(B)
            assert stt == ores.OK
            sl = np.asarray(slots)
            assert [(int(res.sim[j]), int(res.t[j])) for j in sl] == [recs[i][:2] for i in b]
            xn = mlp.normalise_inputs(res.X[sl], res.t[sl], tau)
            tn = ores.stored_to_f64(res.payload[sl], cfg.storage)
            loss, p, m, v, _ = otr.one_step_from_state(p, m, v, k, S, [(xn, tn)], n)
            k, S = k + 1, S + B
            losses_o.append(loss)
        got = np.asarray(losses_g)
        ref = np.asarray(losses_o[-steps:])
        tol = 1e-5 if precision == mel.FP32 else 2e-2
        assert np.max(np.abs(got - ref) / ref) <= tol, (got, ref)
    after = ctx.get_state()
    assert after["k"] == k and after["S"] == S
    if precision == mel.FP32:
        assert max(rel_norm(a, b) for a, b in zip(tensors_f64(after["p"]), p)) <= 1e-5
    ds.close()


def test_offline_dataset_smaller_than_a_batch(tmp_path):
    """count < B: no full batch in an epoch (the partial tail is dropped, R24) -> 0 steps."""
    n, B = 100, 16
    recs = _records(1, 10, n)
    path = str(tmp_path / "small.bin")
    mel.write_dataset(path, n, recs)
    ds = mel.Dataset(path, threads=2)
    ctx = mel.Context(mel.Config(n_field=n, hidden=(32,), capacity=2 * B, threshold=0, batch=B, steps_per_sim=10,
                                 staging_entries=2 * B, policy=mel.FIFO))
    steps, losses = ctx.train_offline(ds, seed=1, epoch=0)
    assert steps == 0 and len(losses) == 0
    assert ctx.get_state()["k"] == 0
    ds.close()
