"""GPU parity of the reservoir path (Alg. 1) and of the fp32 training
step, through the C ABI, against the oracle on the same seeded op-logs.
Bar: reservoir contents, sampled slots and counters bit-exact; fp32-mode loss and
per-tensor weights within 1e-5 relative (re-anchored, BASELINE north_star)."""
import random
from dataclasses import replace

import numpy as np
import pytest

from mel_inputs import design
from oracle import mlp, reservoir as ores

from harness import FieldTable, compare_reservoir, make_config, replay_parity

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mel():
    from paper_2309_16743_b200 import build, mel as m
    build.build()
    return m


@pytest.mark.parametrize("wl", [design.TINY, design.MEDIUM], ids=["tiny", "medium"])
def test_init_params_bit_exact(mel, wl):
    ctx = mel.Context(make_config(replace(wl, capacity=512, threshold=100)))
    got = ctx.get_params()
    want = [x for Wb in mlp.init_params(mlp.layer_dims(wl.n_field, wl.hidden), seed=1) for x in Wb]
    for g, w in zip(got, want):
        assert np.array_equal(g.reshape(-1).view(np.uint32), w.reshape(-1).view(np.uint32))


@pytest.mark.parametrize("wl,storage", [(design.TINY, 0), (design.TINY_EVICT, 0), (design.TINY_EVICT, 1)],
                         ids=["tiny-f32", "tiny_evict-f32", "tiny_evict-bf16store"])
def test_tiny_oplog_to_eos_reanchored(mel, wl, storage):
    table = FieldTable(wl)
    ctx = mel.Context(make_config(wl, storage=storage))
    rep = replay_parity(ctx, wl, table, design.build_oplog(wl), storage=storage)
    res = rep["oracle_res"]
    assert res.over and res.p == 0, "replay must reach EOS"
    compare_reservoir(ctx, res, storage)
    assert rep["steps"] > 20
    assert max(rep["loss_err"]) <= 1e-5, max(rep["loss_err"])
    assert max(rep["w_err"]) <= 1e-5, max(rep["w_err"])
    if wl.capacity < wl.sims * wl.tau:
        assert res.evictions > 0


def test_medium_geometry_with_evictions_reanchored(mel):
    wl = replace(design.MEDIUM, name="medium-evict", capacity=2000, threshold=333, sims=60)
    table = FieldTable(wl)
    ctx = mel.Context(make_config(wl))
    ops = design.build_oplog(wl)
    rep = replay_parity(ctx, wl, table, ops, max_train_steps=25)
    compare_reservoir(ctx, rep["oracle_res"])
    assert rep["oracle_res"].evictions > 0
    assert max(rep["loss_err"]) <= 1e-5 and max(rep["w_err"]) <= 1e-5, (max(rep["loss_err"]), max(rep["w_err"]))
    assert max(rep["tile_err"]) <= 1e-5, max(rep["tile_err"])


@pytest.mark.slow
def test_medium_config_fp32_1000_steps_reanchored(mel):
    """SURVEY 8(c) O7 at BASELINE configs[1] as stated: medium (100x100 grid, tau 100, 1000
    sims, 6-256-256-10^4, C = 50,000, theta = 8,333, B = 256), fp32 mode, every one of 1000
    training steps re-anchored to the fp64 oracle step (loss and every tensor <= 1e-5, W_L per
    128-row tile <= 1e-5, north star); sampled slots bit-exact on every SAMPLE."""
    wl = design.MEDIUM
    table = FieldTable(wl)
    ctx = mel.Context(make_config(wl))
    rep = replay_parity(ctx, wl, table, design.build_oplog(wl), max_train_steps=1000)
    print("medium fp32: %d steps, loss err %.2e, w err %.2e, W_L tile err %.2e, max abs %.2e" %
          (rep["steps"], max(rep["loss_err"]), max(rep["w_err"]), max(rep["tile_err"]), max(rep["max_abs"])))
    assert rep["steps"] == 1000
    assert max(rep["loss_err"]) <= 1e-5 and max(rep["w_err"]) <= 1e-5 and max(rep["tile_err"]) <= 1e-5


@pytest.mark.parametrize("seed", [3, 4])
def test_random_schedules_with_backpressure_and_ring_wrap(mel, seed):
    """Random interleavings (bursty producer, small C so that u == C back-pressure
    happens, staging ring of 6 entries so reservoir_put returns EAGAIN), no
    training: slots and final contents bit-exact."""
    wl = replace(design.TINY, capacity=8, threshold=2, batch=2)
    table = FieldTable(wl)
    ctx = mel.Context(make_config(wl, staging=6, seed=seed))
    res = ores.Reservoir(wl.capacity, wl.threshold, wl.n_field, seed=seed)
    rng = random.Random(seed)
    order = design.stream_order(wl.sims, wl.tau)
    i = 0
    backpressure = ring_full = 0
    while i < len(order):
        for _ in range(rng.randrange(14)):
            if i >= len(order):
                break
            s, t = order[i]
            r = ctx.put(s, t, table.Xs(s), table.field(s, t))
            if r == 1:
                ring_full += 1
                break
            res.put(s, t, table.Xs(s), table.field(s, t))
            i += 1
        st_o, sl_o = res.sample(wl.batch)
        st_g, sl_g, n = ctx.sample(want_slots=True)
        assert st_o == st_g and list(sl_g) == list(sl_o)
        backpressure += int(len(res.pend) > 0)
        ctx.step(want_loss=False) if st_g == 0 else None
    ctx.close(); res.close()
    while True:
        st_o, sl_o = res.sample(wl.batch)
        st_g, sl_g, n = ctx.sample(want_slots=True)
        assert list(sl_g) == list(sl_o)
        if not sl_o:
            break
    compare_reservoir(ctx, res)
    assert backpressure > 0 and ring_full > 0
    with pytest.raises(mel.MelError) as e:
        ctx.put(0, 0, table.Xs(0), table.field(0, 0))
    assert e.value.code == mel.ECLOSED
    with pytest.raises(mel.MelError) as e:
        ctx.close()
    assert e.value.code == mel.EPROTO


@pytest.mark.parametrize("offset,zc", [(0, True), (1, True), (0, False)],
                         ids=["zero-copy", "unaligned-copied", "copied"])
def test_device_resident_puts_match_host_puts(mel, offset, zc):
    """Device puts: with zero_copy an aligned field is read by the commit straight from the
    caller's buffer (field_on_device 2); a 4-byte-offset one, or any without zero_copy, is
    copied at the call.  All must equal the host puts bit for bit."""
    import torch
    wl = design.TINY_EVICT
    table = FieldTable(wl)
    a = mel.Context(make_config(wl))
    b = mel.Context(make_config(wl))
    keep = []    # device sources must stay alive until the library's stream read them
    for (s, t) in design.stream_order(wl.sims, wl.tau)[:60]:
        f = table.field(s, t)
        a.put(s, t, table.Xs(s), f)
        buf = torch.zeros(len(f) + offset, dtype=torch.float32, device="cuda")
        buf[offset:] = torch.from_numpy(f).cuda()
        keep.append(buf)
        torch.cuda.synchronize()
        b.put(s, t, table.Xs(s), buf[offset:], zero_copy=zc)
        if t % 5 == 4:
            assert list(a.sample(True)[1]) == list(b.sample(True)[1])
    da, db = a.dump(), b.dump()
    for k in da:
        assert np.array_equal(da[k], db[k]), k


def test_copied_device_put_buffer_reusable_after_the_call(mel):
    """field_on_device 1 (the default for torch tensors): the field is copied on the
    context's stream at the call, so the caller may overwrite its buffer right after
    (same stream order) -- the reservoir still holds the values put."""
    import torch
    wl = replace(design.TINY, capacity=16, threshold=2, batch=4)
    table = FieldTable(wl)
    stream = torch.cuda.Stream()
    a = mel.Context(make_config(wl))
    b = mel.Context(make_config(wl), stream=stream.cuda_stream)   # the producer's stream
    with torch.cuda.stream(stream):
        buf = torch.zeros(wl.n_field, dtype=torch.float32, device="cuda")
        for (s, t) in design.stream_order(wl.sims, wl.tau)[:12]:
            f = table.field(s, t)
            a.put(s, t, table.Xs(s), f)
            buf.copy_(torch.from_numpy(f).cuda())
            b.put(s, t, table.Xs(s), buf)
            buf.fill_(float("nan"))             # reused before any commit has run
    a.sample(); b.sample()
    da, db = a.dump(), b.dump()
    for k in da:
        assert np.array_equal(da[k], db[k]), k


def test_degenerate_capacity_one_threshold_zero(mel):
    """C = 1, theta = 0, B = 1: every put after the first must wait for the single
    item to be seen, and each commit evicts it; trained to EOS."""
    wl = replace(design.TINY, capacity=1, threshold=0, batch=1, puts_per_step=2, sims=4)
    table = FieldTable(wl)
    ctx = mel.Context(make_config(wl, staging=64))   # back-pressure keeps up to 40 puts pending
    rep = replay_parity(ctx, wl, table, design.build_oplog(wl, n_steps_after_close=60))
    res = rep["oracle_res"]
    compare_reservoir(ctx, res)
    assert res.evictions > 0 and rep["steps"] > 10
    assert max(rep["loss_err"]) <= 1e-5 and max(rep["w_err"]) <= 1e-5
