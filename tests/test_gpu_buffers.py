"""GPU parity of the FIFO and FIRO comparison buffers (PAPER.md P:221-223,
reading R21) through the C ABI against the oracle on the same seeded op-logs:
sampled slots, statuses, buffer contents and counters bit-exact; the training
steps fed by them re-anchored within the fp32 / bf16 bars of DESIGN.md §3."""
import random
from dataclasses import replace

import pytest

from mel_inputs import design
from oracle import reservoir as ores

from harness import FieldTable, compare_reservoir, make_config, replay_parity

pytestmark = pytest.mark.gpu
POLICIES = [(ores.FIFO, "fifo"), (ores.FIRO, "firo")]


@pytest.fixture(scope="module")
def mel():
    from paper_2309_16743_b200 import build, mel as m
    build.build()
    return m


@pytest.mark.parametrize("policy,name", POLICIES, ids=[n for _, n in POLICIES])
@pytest.mark.parametrize("wl,storage", [(design.TINY, 0), (design.TINY_EVICT, 1)], ids=["tiny-f32", "tiny_evict-bf16store"])
def test_tiny_oplog_to_eos(mel, policy, name, wl, storage):
    table = FieldTable(wl)
    ctx = mel.Context(make_config(wl, storage=storage, policy=policy))
    rep = replay_parity(ctx, wl, table, design.build_oplog(wl), storage=storage, policy=policy)
    res = rep["oracle_res"]
    assert res.over and res.p == 0
    compare_reservoir(ctx, res, storage)
    # every accepted item is seen exactly once ("seen once, and only once")
    assert rep["samples"] == res.accepted and res.hist[1] == res.accepted
    assert max(rep["loss_err"]) <= 1e-5 and max(rep["w_err"]) <= 1e-5, (max(rep["loss_err"]), max(rep["w_err"]))


@pytest.mark.parametrize("policy,name", POLICIES, ids=[n for _, n in POLICIES])
def test_medium_bf16_training(mel, policy, name):
    wl = replace(design.MEDIUM, name="medium-bf16-" + name, capacity=600, threshold=100, sims=20, batch=128,
                 puts_per_step=100)
    table = FieldTable(wl)
    ctx = mel.Context(make_config(wl, precision=1, storage=1, policy=policy))
    rep = replay_parity(ctx, wl, table, design.build_oplog(wl), storage=1, max_train_steps=6, policy=policy)
    assert rep["steps"] == 6
    assert max(rep["loss_err"]) <= 2e-2 and max(rep["w_err"]) <= 1e-3, (max(rep["loss_err"]), max(rep["w_err"]))
    compare_reservoir(ctx, rep["oracle_res"], 1)


@pytest.mark.parametrize("policy,name", POLICIES, ids=[n for _, n in POLICIES])
@pytest.mark.parametrize("seed", [3, 4])
def test_random_schedules_full_buffer_and_ring(mel, policy, name, seed):
    """Bursty producer, C = 8 so that a full buffer suspends production, staging
    ring of 6 entries so reservoir_put returns EAGAIN; to EOS, no training."""
    wl = replace(design.TINY, capacity=8, threshold=2, batch=3)
    table = FieldTable(wl)
    ctx = mel.Context(make_config(wl, staging=6, seed=seed, policy=policy))
    res = ores.Reservoir(wl.capacity, wl.threshold, wl.n_field, seed=seed, policy=policy)
    rng = random.Random(seed)
    order = design.stream_order(wl.sims, wl.tau)
    i = suspended = ring_full = eagain = 0
    while i < len(order):
        for _ in range(rng.randrange(10)):
            if i >= len(order):
                break
            s, t = order[i]
            if ctx.put(s, t, table.Xs(s), table.field(s, t)) == 1:
                ring_full += 1
                break
            res.put(s, t, table.Xs(s), table.field(s, t))
            i += 1
        if rng.random() < 0.3:
            continue                                   # consumer pause: the buffer fills
        st_o, sl_o = res.sample(wl.batch)
        st_g, sl_g, n = ctx.sample(want_slots=True)
        assert st_o == st_g and list(sl_g) == list(sl_o)
        eagain += int(st_o == ores.EAGAIN)
        suspended += int(len(res.pend) > 0)
        ctx.step(want_loss=False) if st_g == 0 else None
    ctx.close(); res.close()
    while True:
        st_o, sl_o = res.sample(wl.batch)
        st_g, sl_g, n = ctx.sample(want_slots=True)
        assert list(sl_g) == list(sl_o)
        if not sl_o:
            break
    compare_reservoir(ctx, res)
    assert suspended > 0 and ring_full > 0
    assert res.hist[1] == res.accepted == len(order)


def test_invalid_policy_configs(mel):
    wl = replace(design.TINY, capacity=8, threshold=2, batch=9)
    with pytest.raises(mel.MelError):
        mel.Context(make_config(wl, policy=ores.FIFO))          # B > C
    with pytest.raises(mel.MelError):
        mel.Context(make_config(replace(wl, batch=7), policy=ores.FIRO))   # theta + B > C
    with pytest.raises(mel.MelError):
        mel.Context(make_config(wl, policy=3))
