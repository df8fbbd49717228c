"""GPU parity of the training step in bf16 mode (tcgen05 output layer) and of
validation, against the oracle.  Tolerances: DESIGN.md "Parity bars"."""
from dataclasses import replace

import numpy as np
import pytest

from mel_inputs import design
from oracle import mlp, reservoir as ores, trainer as otr

from harness import FieldTable, make_config, rel_norm, replay_parity, tensors_f64

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mel():
    from paper_2309_16743_b200 import build, mel as m
    build.build()
    return m


def _bf16_wl(**kw):
    base = replace(design.MEDIUM, name="medium-bf16", capacity=2000, threshold=333, sims=60)
    return replace(base, **kw)


@pytest.mark.parametrize("n,batch,flags", [(100, 256, 0), (37, 64, 0), (101, 192, 0), (100, 256, 8), (100, 10, 0),
                                          (37, 100, 0), (37, 300, 0)],
                         ids=["N1e4-B256", "N1369-B64", "N10201-B192", "N1e4-B256-unfusedAdam", "N1e4-B10-paper",
                              "N1369-B100", "N1369-B300-fused-padded"])
def test_bf16_step_reanchored(mel, n, batch, flags):
    """One re-anchored bf16 step at a time: the GPU's output layer runs on
    tcgen05 with bf16 operands (W shadow, H, dY) and fp32 TMEM accumulation.
    Sizes span several 128-row tiles, ragged tails (N % 128 != 0), B not a multiple of
    128, and B not a multiple of 64 (10 = the paper's per-GPU batch; 100): the
    kernels run the batch padded to whole 64-row chunks with the padding rows masked."""
    wl = _bf16_wl(n=n, batch=batch, hidden=(256, 256))
    table = FieldTable(wl)
    ctx = mel.Context(make_config(wl, precision=1, storage=1, flags=flags))
    rep = replay_parity(ctx, wl, table, design.build_oplog(wl), storage=1, max_train_steps=6)
    print("bf16 re-anchored: loss err %.3e  weight err %.3e  W_L tile err %.3e" %
          (max(rep["loss_err"]), max(rep["w_err"]), max(rep["tile_err"])))
    assert rep["steps"] == 6
    assert max(rep["loss_err"]) <= 2e-2
    assert max(rep["w_err"]) <= 1e-3
    assert max(rep["tile_err"]) <= 5e-3


@pytest.mark.slow
def test_bf16_loss_after_1000_steps_free_running(mel):
    """north_star: <= 2e-2 relative loss at step 1000 in bf16 mode (same batches,
    free-running from the same init)."""
    wl = replace(design.MEDIUM, name="medium-1k", capacity=6000, threshold=1000, sims=1100, puts_per_step=100)
    table = FieldTable(wl)
    ctx = mel.Context(make_config(wl, precision=1, storage=1))
    tr = otr.Trainer(wl.n_field, wl.hidden, wl.tau, wl.capacity, wl.threshold, wl.batch, seed=1, storage=1)
    losses_g, losses_o = [], []
    for op in design.build_oplog(wl):
        if op[0] == "PUT":
            _, r, s, t = op
            ctx.put(s, t, table.Xs(s), table.field(s, t)); tr.put(0, s, t, table.Xs(s), table.field(s, t))
        elif op[0] == "SAMPLE":
            a = ctx.sample()[0]; b = tr.sample(0)[0]
            assert a == b
        elif op[0] == "STEP":
            a, lg = ctx.step(want_loss=True)
            b, lo = tr.step()
            assert a == b
            if a == 0:
                losses_g.append(lg); losses_o.append(lo)
                if len(losses_g) == 1000:
                    break
    assert len(losses_g) == 1000
    err = abs(losses_g[-1] - losses_o[-1]) / losses_o[-1]
    tail = np.mean(np.abs(np.array(losses_g[-50:]) - np.array(losses_o[-50:])) / np.array(losses_o[-50:]))
    print("bf16 step-1000 loss rel err %.3e (mean over 951-1000: %.3e); loss %.4e -> %.4e" %
          (err, tail, losses_o[0], losses_o[-1]))
    assert err <= 2e-2


@pytest.mark.parametrize("hidden,batch,overlap", [((256, 256), 256, False), ((64, 64), 320, False),
                                                  ((256, 256), 256, True), ((64, 64), 320, True),
                                                  ((256, 256), 10, False), ((256, 256), 64, False)],
                         ids=["K256-B256", "K64-B320-padded", "K256-B256-overlapped", "K64-B320-overlapped",
                              "K256-B10-paper", "K256-B64"])
def test_fused_adam_bit_identical_to_unfused(mel, hidden, batch, overlap, monkeypatch):
    """Adam of W_L inside the output-layer kernel (default at world 1, bf16, B >= 256)
    reproduces the separate Adam kernel bit for bit (master, moments, shadow) over 40
    free-running steps: same arithmetic, only where it runs differs -- in the
    staged K1 and in the opt-in overlapped K1 (MEL_K1_OVERLAP=1: Adam CTAs fed through the
    L2 ring).  N = 10^4 + 37 leaves a ragged last tile; B = 320 runs padded to 384."""
    wl = _bf16_wl(n=101, batch=batch, hidden=hidden, capacity=600, threshold=100, sims=40, puts_per_step=40)
    table = FieldTable(wl)
    states = []
    for flags in (0, mel.FLAG_UNFUSED_ADAM):
        monkeypatch.setenv("MEL_K1_OVERLAP", "1" if (overlap and flags == 0) else "0")
        ctx = mel.Context(make_config(wl, precision=1, storage=1, flags=flags))
        steps = 0
        for op in design.build_oplog(wl):
            if op[0] == "PUT":
                _, r, s, t = op
                ctx.put(s, t, table.Xs(s), table.field(s, t))
            elif op[0] == "CLOSE":
                ctx.close()
            elif op[0] == "SAMPLE":
                ctx.sample()
            elif op[0] == "STEP":
                if ctx.step()[0] == 0:
                    steps += 1
                    if steps == 40:
                        break
        assert steps == 40
        st = ctx.get_state()
        states.append(st)
    a, b = states
    for name in ("p", "m", "v"):
        for x, y in zip(a[name], b[name]):
            assert np.array_equal(x.view(np.uint32), y.view(np.uint32)), name


@pytest.mark.parametrize("batch,flags,hidden,overlap", [(256, 0, (256, 256), 0), (320, 0, (256, 256), 0),
                                                       (128, 8, (256, 256), 0), (448, 0, (128, 128), 0),
                                                       (300, 0, (128, 64), 0), (320, 0, (256, 256), 1),
                                                       (10, 0, (256, 256), 0)],
                         ids=["fused-adam", "fused-adam-5-chunks", "unfused-adam", "K128-7-chunks", "K64-B300-padded",
                              "overlapped-5-chunks", "fused-B10-1-chunk"])
def test_k1_result_independent_of_grid(mel, batch, flags, hidden, overlap, monkeypatch):
    """Race canary for K1's barrier protocols (compute-sanitizer is not
    available on this pool): each 128-row tile's forward, gradient and fused Adam depend only
    on the tile, so the persistent grid's size must not change a single bit of p, m, v.  A
    grid of 148, 29, 7 or 1 CTA(s) walks every mbarrier ring (H chunks, targets, Y/dY TMEM
    buffers, Adam stages, early W) through a different phase pattern per CTA (2..79 tiles
    each); a missed wait or a wrong parity shows up as a difference (or a trap), 25 steps.
    B = 320 runs 5 chunks per tile, so the target ring's phase shifts from tile to tile: the
    next tile's targets must not land in the slots the fused Adam still stages in (a bug
    until round 2's end, invisible at <= 1 tile per CTA)."""
    wl = _bf16_wl(n=101, batch=batch, hidden=hidden, capacity=600, threshold=100, sims=40, puts_per_step=40)
    table = FieldTable(wl)
    states = []
    # overlapped variant (opt-in): MMA CTAs hand dW tiles to Adam CTAs through two ring slots
    # each -- at 7 CTAs (5 MMA + 2 Adam) every MMA CTA recycles its slots many times
    monkeypatch.setenv("MEL_K1_OVERLAP", str(overlap))
    for ctas in (0, 29, 7, 2) if overlap else (0, 29, 7, 1):
        if ctas:
            monkeypatch.setenv("MEL_K1_CTAS", str(ctas))
        else:
            monkeypatch.delenv("MEL_K1_CTAS", raising=False)
        ctx = mel.Context(make_config(wl, precision=1, storage=1, flags=flags))
        steps = 0
        for op in design.build_oplog(wl):
            if op[0] == "PUT":
                _, r, s, t = op
                ctx.put(s, t, table.Xs(s), table.field(s, t))
            elif op[0] == "CLOSE":
                ctx.close()
            elif op[0] == "SAMPLE":
                ctx.sample()
            elif op[0] == "STEP":
                if ctx.step()[0] == 0:
                    steps += 1
                    if steps == 25:
                        break
        assert steps == 25
        states.append(ctx.get_state())
    for st in states[1:]:
        for name in ("p", "m", "v"):
            for x, y in zip(states[0][name], st[name]):
                assert np.array_equal(x.view(np.uint32), y.view(np.uint32)), name


@pytest.mark.parametrize("precision", [0, 1])
def test_eval_matches_oracle(mel, precision):
    wl = _bf16_wl(n=40, batch=128)
    table = FieldTable(wl)
    ctx = mel.Context(make_config(wl, precision=precision, storage=precision))
    Xv = design.draw_design(3, seed=1, validation=True)
    from mel_inputs import heat
    fields = np.concatenate([heat.simulate(Xv[i], wl.n, wl.tau) for i in range(3)])
    X = np.repeat(Xv, wl.tau, axis=0)
    t = np.tile(np.arange(wl.tau), 3).astype(np.uint32)
    mse, pred = ctx.eval(X, t, fields, want_pred=True)
    params = [(W.astype(np.float64), b.astype(np.float64)) for W, b in mlp.unflatten(ctx.get_params())]
    xn = mlp.normalise_inputs(X, t, wl.tau)
    tn = ores.normalise_f32(fields).astype(np.float64)
    want = mlp.mse(params, xn, tn)
    assert abs(mse - want) / want < 1e-5
    Y = mlp.forward(params, xn)[1][-1] * 400.0 + 100.0
    assert np.max(np.abs(pred - Y)) < 1e-2


def test_bf16_to_eos_with_short_drain_batches(mel):
    """bf16 path through reception, close and drain (batches shorter than B, then
    EOS); hidden 64x64 exercises the K = 64 instantiation of the tensor-core kernels."""
    wl = replace(design.MEDIUM, name="bf16-eos", n=16, tau=10, sims=12, hidden=(64, 64), capacity=48, threshold=8,
                 batch=64, puts_per_step=20)
    table = FieldTable(wl)
    ctx = mel.Context(make_config(wl, precision=1, storage=1))
    rep = replay_parity(ctx, wl, table, design.build_oplog(wl), storage=1)
    res = rep["oracle_res"]
    assert res.over and res.p == 0
    assert rep["samples"] % wl.batch != 0            # at least one short drain batch
    assert max(rep["loss_err"]) <= 2e-2 and max(rep["w_err"]) <= 1e-3, (max(rep["loss_err"]), max(rep["w_err"]))


@pytest.mark.parametrize("hidden,batch", [((128,), 128), ((256, 256), 2048)], ids=["one-hidden-K128", "B2048"])
def test_bf16_shapes(mel, hidden, batch):
    wl = _bf16_wl(n=64, batch=batch, hidden=hidden, capacity=4096, threshold=2048, sims=80, puts_per_step=1000)
    table = FieldTable(wl)
    ctx = mel.Context(make_config(wl, precision=1, storage=1))
    rep = replay_parity(ctx, wl, table, design.build_oplog(wl), storage=1, max_train_steps=3)
    assert rep["steps"] == 3
    assert max(rep["loss_err"]) <= 2e-2 and max(rep["w_err"]) <= 1e-3, (max(rep["loss_err"]), max(rep["w_err"]))


def test_invalid_configurations_fail_loudly(mel):
    base = dict(n_field=400, hidden=(256, 256), capacity=100, threshold=10, batch=128, precision=1, storage=1)
    for bad in (dict(threshold=100), dict(batch=0), dict(hidden=(256, 100)), dict(storage=0),
                dict(n_field=0)):
        cfg = mel.Config(**{**base, **bad})
        with pytest.raises(mel.MelError) as e:
            mel.Context(cfg)
        assert e.value.code == mel.EINVAL


def test_step_result_matches_synchronous_loss(mel):
    """surrogate_step_result(i) returns the same loss as the synchronous
    surrogate_step(loss) of that call, for the last 16 calls, without a stream drain."""
    wl = _bf16_wl(n=40, batch=128, capacity=400, threshold=50, sims=30, puts_per_step=40)
    table = FieldTable(wl)
    a = mel.Context(make_config(wl, precision=1, storage=1))
    b = mel.Context(make_config(wl, precision=1, storage=1))
    sync_losses, calls = [], 0
    for op in design.build_oplog(wl):
        if op[0] == "PUT":
            _, r, s, t = op
            a.put(s, t, table.Xs(s), table.field(s, t)); b.put(s, t, table.Xs(s), table.field(s, t))
        elif op[0] == "SAMPLE":
            a.sample(); b.sample()
        elif op[0] == "STEP":
            st_a, la = a.step(want_loss=True)
            st_b, _ = b.step(want_loss=False)
            sync_losses.append((st_a, la))
            calls += 1
            if calls == 20:
                break
    for i in range(calls - 16, calls):
        st, loss = b.step_result(i)
        st_a, la = sync_losses[i]
        assert st == (0 if st_a == 0 else 1)
        if st_a == 0:
            assert loss == la
    with pytest.raises(mel.MelError):
        b.step_result(calls - 17)
    with pytest.raises(mel.MelError):
        b.step_result(calls)


@pytest.mark.parametrize("precision", [0, 1])
def test_fused_head_matches_generic_head(mel, precision, monkeypatch):
    """The fused head kernels (forward: one launch for the gather, both hidden layers and the
    step scalars; backward: per-block partials + one fixed-order reduction launch that also
    finalises the step at world 1) against the generic per-GEMM head path (MEL_HEAD_FUSED=0,
    split-K SGEMMs, separate gather / prepare / reduce / finalize kernels) over 30
    free-running steps: the sums are grouped differently, so losses and parameters agree to
    fp32 rounding."""
    wl = _bf16_wl(n=37, batch=320, hidden=(256, 256), capacity=600, threshold=100, sims=40, puts_per_step=40)
    table = FieldTable(wl)
    states, losses = [], []
    for fused in ("1", "0"):
        monkeypatch.setenv("MEL_HEAD_FUSED", fused)
        ctx = mel.Context(make_config(wl, precision=precision, storage=precision))
        steps, ls = 0, []
        for op in design.build_oplog(wl):
            if op[0] == "PUT":
                _, r, s, t = op
                ctx.put(s, t, table.Xs(s), table.field(s, t))
            elif op[0] == "SAMPLE":
                ctx.sample()
            elif op[0] == "STEP":
                rc, lo = ctx.step(want_loss=True)
                if rc == 0:
                    steps += 1
                    ls.append(lo)
                    if steps == 30:
                        break
        assert steps == 30
        states.append(ctx.get_state())
        losses.append(np.array(ls))
    assert abs(losses[0][0] - losses[1][0]) <= 1e-6 * losses[1][0]   # first step: forward only
    assert np.max(np.abs(losses[0] - losses[1]) / losses[1]) <= 1e-4
    for x, y in zip(states[0]["p"], states[1]["p"]):
        assert rel_norm(x, y) <= (1e-5 if precision == 0 else 1e-3)   # bf16: H2 rounding flips compound
