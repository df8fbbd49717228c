"""Pins for oracle/mlp.py and oracle/trainer.py: finite differences, special
cases, Adam and LR closed forms, the data-parallel identity, and a
training-sanity check.  Cited lines: PAPER.md P:171-173, P:308, P:362, P:371;
SPEC.md S:243-294 for the example values."""
import numpy as np
import pytest

from oracle import mlp, trainer


def _toy(dims, seed=0, B=5):
    rng = np.random.default_rng(seed)
    params = [(rng.normal(0, 0.5, (dims[l + 1], dims[l])), rng.normal(0, 0.1, dims[l + 1]))
              for l in range(len(dims) - 1)]
    xn = rng.uniform(0, 1, (B, dims[0]))
    tn = rng.uniform(0, 1, (B, dims[-1]))
    return params, xn, tn


@pytest.mark.parametrize("dims", [[6, 8, 4], [6, 5, 7, 3]])
def test_gradients_match_central_finite_differences(dims):
    params, xn, tn = _toy(dims)
    loss, grads = mlp.loss_and_grads(params, xn, tn)
    h = 1e-6
    for l, (W, b) in enumerate(params):
        for arr, g in ((W, grads[l][0]), (b, grads[l][1])):
            it = np.nditer(arr, flags=["multi_index"])
            for _ in it:
                i = it.multi_index
                old = arr[i]
                arr[i] = old + h; lp = mlp.mse(params, xn, tn)
                arr[i] = old - h; lm = mlp.mse(params, xn, tn)
                arr[i] = old
                fd = (lp - lm) / (2 * h)
                assert abs(fd - g[i]) <= 1e-7 * max(1.0, abs(fd)) + 1e-9, (l, i, fd, g[i])


def test_special_cases():
    dims = [6, 8, 4]
    params, xn, tn = _toy(dims)
    zero = [(np.zeros_like(W), np.zeros_like(b)) for W, b in params]
    assert np.all(mlp.forward(zero, xn)[1][-1] == 0)
    one = [(np.zeros((2, 1)), np.zeros(2))]
    assert mlp.mse(one, np.ones((1, 1)), np.array([[-1.0, -2.0]])) == 2.5    # S:253 MSE([1,2],[0,0])
    Y = mlp.forward(params, xn)[1][-1]
    loss, g = mlp.loss_and_grads(params, xn, Y)
    assert loss == 0 and all(np.all(gw == 0) and np.all(gb == 0) for gw, gb in g)
    l1, g1 = mlp.loss_and_grads(params, xn, tn)
    l2, g2 = mlp.loss_and_grads(params, np.vstack([xn, xn]), np.vstack([tn, tn]))
    assert abs(l1 - l2) < 1e-15
    for (a, b), (c, d) in zip(g1, g2):
        np.testing.assert_allclose(a, c, rtol=1e-13); np.testing.assert_allclose(b, d, rtol=1e-13)


def test_relu_derivative_at_zero_is_zero():
    W1 = np.array([[1.0, -1.0]]); b1 = np.array([0.0])       # z = x0 - x1 = 0
    params = [(W1, b1), (np.array([[2.0]]), np.array([0.0]))]
    _, g = mlp.loss_and_grads(params, np.array([[0.3, 0.3]]), np.array([[1.0]]))
    assert np.all(g[0][0] == 0) and np.all(g[0][1] == 0)


def test_adam_closed_forms():
    # step 1 from zero moments: dp = -lr * g / (|g| + eps)
    p, m, v = mlp.adam_update(np.array([0.0]), np.array([1.0]), np.zeros(1), np.zeros(1), 1, 1e-3)
    assert abs(p[0] - (-1e-3 * 1.0 / (1.0 + 1e-8))) < 1e-18
    assert abs(p[0] + 9.9999999e-4) < 1e-12
    # zero gradient: parameters unchanged, moments decayed
    p, m2, v2 = mlp.adam_update(np.array([0.5]), np.array([0.0]), np.array([0.2]), np.array([0.3]), 5, 1e-3)
    assert abs(m2[0] - 0.18) < 1e-15 and abs(v2[0] - 0.3 * 0.999) < 1e-15
    # with non-zero moments the parameter still moves by -lr*mhat/(sqrt(vhat)+eps)
    assert p[0] < 0.5
    # constant gradient g: after k steps mhat = vhat^(1/2) = |g| exactly (bias correction)
    pp, mm, vv = np.array([0.0]), np.zeros(1), np.zeros(1)
    for k in range(1, 6):
        pp, mm, vv = mlp.adam_update(pp, np.array([2.0]), mm, vv, k, 1e-3)
    assert abs(pp[0] + 5 * 1e-3 * 2.0 / (2.0 + 1e-8)) < 1e-15


@pytest.mark.parametrize("S,lr", [(0, 1e-3), (9216, 1e-3), (9999, 1e-3), (10000, 5e-4),
                                  (10240, 5e-4), (20480, 2.5e-4), (40000, 2.5e-4), (10**9, 2.5e-4)])
def test_lr_schedule_values(S, lr):
    # P:371 "halved every 10,000 training samples until it reaches a minimum of 2.5E-4"
    assert mlp.lr_schedule(S) == lr


def test_init_range_and_layout():
    dims = mlp.layer_dims(100, (32,))
    assert dims == [6, 32, 100] and mlp.n_params(dims) == 3524
    assert mlp.n_params(mlp.layer_dims(10**6, (256, 256))) == 257_067_584   # P:308 shapes (Q14)
    p = mlp.init_params(dims, seed=1)
    for l, (W, b) in enumerate(p):
        a = 1 / np.sqrt(dims[l])
        assert W.shape == (dims[l + 1], dims[l]) and W.dtype == np.float32
        assert np.abs(W).max() <= np.float32(a) and np.abs(b).max() <= np.float32(a)
        assert abs(W.mean()) < 0.1 * a
    p2 = mlp.init_params(dims, seed=2)
    assert not np.array_equal(p[0][0], p2[0][0])


def test_data_parallel_step_equals_union_batch():
    # all-reduced gradient of R ranks == gradient of the union batch when
    # all ranks contribute (rank-ordered concatenation), to fp64 rounding.
    dims = [6, 7, 9]
    params, _, _ = _toy(dims)
    rng = np.random.default_rng(1)
    batches = [(rng.uniform(0, 1, (4, 6)), rng.uniform(0, 1, (4, 9))) for _ in range(3)]
    tensors = mlp.flatten(params)
    loss_r, g_r = trainer.global_loss_and_grads(tensors, batches, 9)
    xu = np.vstack([b[0] for b in batches]); tu = np.vstack([b[1] for b in batches])
    loss_1, g_1 = mlp.loss_and_grads(params, xu, tu)
    assert abs(loss_r - loss_1) <= 1e-12 * loss_1
    for a, b in zip(g_r, mlp.flatten(g_1)):
        np.testing.assert_allclose(a, b, rtol=1e-12, atol=1e-15)
    # and the mean of per-rank means (DDP) when every n_r is equal
    means = [mlp.loss_and_grads(params, x, t) for x, t in batches]
    for i, a in enumerate(g_r):
        ddp = sum(mlp.flatten(g)[i] for _, g in means) / 3
        np.testing.assert_allclose(a, ddp, rtol=1e-12, atol=1e-15)


def test_training_reduces_loss_tenfold():
    # S:294 sanity: 500 Adam steps on a fixed 100-sample toy regression
    rng = np.random.default_rng(0)
    dims = [6, 32, 20]
    xn = rng.uniform(0, 1, (100, 6))
    tn = np.tanh(xn @ rng.normal(0, 1, (6, 20)))
    tensors = [x.astype(np.float64) for x in mlp.flatten(mlp.init_params(dims, 3))]
    opt = mlp.Adam(tensors)
    l0 = mlp.mse(mlp.unflatten(tensors), xn, tn)
    for _ in range(500):
        _, g = mlp.loss_and_grads(mlp.unflatten(tensors), xn, tn)
        tensors = opt.step(tensors, mlp.flatten(g), 1e-2)
    assert mlp.mse(mlp.unflatten(tensors), xn, tn) < l0 / 10


def test_trainer_replays_an_oplog_to_eos():
    from mel_inputs import design, heat
    wl = design.TINY_EVICT
    X = design.draw_design(wl.sims, seed=1)
    fields = {s: heat.simulate(X[s], wl.n, wl.tau) for s in range(wl.sims)}
    tr = trainer.Trainer(wl.n_field, wl.hidden, wl.tau, wl.capacity, wl.threshold, wl.batch, seed=1)
    trace = trainer.replay(tr, design.build_oplog(wl), lambda s, t: fields[s][t], lambda s: X[s])
    assert trace["step"][-1][0] == trainer.EOS
    r = tr.res[0]
    assert r.q == wl.sims * wl.tau and r.evictions > 0 and r.p == 0
    losses = [l for st, l in trace["step"] if st == 0]
    assert len(losses) > 10 and losses[-1] < losses[0]
