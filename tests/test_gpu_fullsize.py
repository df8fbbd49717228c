"""Parity at the paper's full size, in the launch configuration bench.py times
(N = 1000x1000 outputs, hidden 256x256, B = 1024, bf16 tcgen05 output layer,
reservoir C = 6000, theta = 1000).  One training step is checked against the
oracle run in fp64 from the GPU's exact pre-step state on the same batch:
  * the global loss (the oracle sweeps all 10^6 outputs in column chunks),
  * every head tensor (their gradients need dS/dH2, a reduction over all N),
  * 512 sampled rows of W3 and b3 (incl. the ragged tail rows),
with the bf16-mode bars of DESIGN.md §3.  The target rows the oracle uses are
the stored-value rule (R17) applied to the same seeded input fields."""
import numpy as np
import pytest

from harness import rel_norm

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def test_paper_shape_one_step_sampled():
    import torch

    from mel_inputs import design, heat_torch
    from oracle import mlp, reservoir as ores
    from paper_2309_16743_b200 import build, mel

    build.build()
    n_grid, tau, B, C, theta = 1000, 100, 1024, 6000, 1000
    N = n_grid * n_grid
    dev = torch.device("cuda", 0)
    ctx = mel.Context(mel.Config(n_field=N, hidden=(256, 256), capacity=C, threshold=theta, batch=B, steps_per_sim=tau,
                                 precision=mel.BF16, storage=mel.STORE_BF16, seed=1, staging_entries=32))
    phi = heat_torch.basis(n_grid, tau, device=dev)
    X = design.draw_design(20, seed=1)
    Xd = torch.from_numpy(X).to(dev)
    order = design.routed_stream(20, tau, 0, 1)[:1100]
    for i in range(0, len(order), 25):
        pairs = order[i:i + 25]
        s = torch.tensor([p[0] for p in pairs], device=dev)
        t = torch.tensor([p[1] for p in pairs], device=dev)
        F = heat_torch.fields(phi, Xd[s], t)
        for j, (ss, tt) in enumerate(pairs):
            assert ctx.put(ss, tt, X[ss], F[j]) == 0
        torch.cuda.synchronize()
        ctx.sample()                     # commit point (EAGAIN until p > theta)
    st, slots, n = ctx.sample(want_slots=True)
    assert st == 0 and n == B
    meta = ctx.dump(payload=False)
    sims, ts = meta["sim"][slots].astype(np.int64), meta["t"][slots].astype(np.int64)
    before = ctx.get_state()
    st, loss_g = ctx.step(want_loss=True)
    assert st == 0
    after = ctx.get_state()

    # ---- oracle step from the same state (fp64) ----
    W1, b1, W2, b2, W3, b3 = [x.astype(np.float64) for x in before["p"]]
    xn = mlp.normalise_inputs(meta["X"][slots], ts, tau)
    Z1 = xn @ W1.T + b1; H1 = np.maximum(Z1, 0)
    Z2 = H1 @ W2.T + b2; H2 = np.maximum(Z2, 0)
    denom = float(B) * N
    sse, dH2 = 0.0, np.zeros_like(H2)
    gW3_rows, gb3_rows = {}, {}
    rng = np.random.default_rng(5)
    sample_rows = np.unique(np.concatenate([rng.choice(N, 500, replace=False), np.arange(N - 12, N)]))
    Xb = torch.from_numpy(meta["X"][slots]).to(dev)
    tb = torch.from_numpy(ts).to(dev)
    chunk = 50_000
    for c0 in range(0, N, chunk):
        c1 = min(N, c0 + chunk)
        F = torch.einsum("kc,ckn->kn", Xb, phi[:, tb, c0:c1]).cpu().numpy()     # same fp32 inputs
        T = ores.stored_to_f64(ores.stored_payload(F, ores.STORE_BF16), ores.STORE_BF16)
        Y = H2 @ W3[c0:c1].T + b3[c0:c1]
        R = Y - T
        sse += float(np.sum(R * R))
        dY = 2.0 * R / denom
        dH2 += dY @ W3[c0:c1]
        rows = sample_rows[(sample_rows >= c0) & (sample_rows < c1)]
        for r in rows:
            gW3_rows[r] = dY[:, r - c0] @ H2
            gb3_rows[r] = dY[:, r - c0].sum()
    loss_o = sse / denom
    dZ2 = dH2 * (Z2 > 0)
    gW2, gb2 = dZ2.T @ H1, dZ2.sum(0)
    dZ1 = (dZ2 @ W2) * (Z1 > 0)
    gW1, gb1 = dZ1.T @ xn, dZ1.sum(0)
    k, S = before["k"] + 1, before["S"]
    lr = mlp.lr_schedule(S)
    m0, v0 = before["m"], before["v"]

    def adam(i, p, g, idx=None):
        mm = m0[i] if idx is None else m0[i][idx]
        vv = v0[i] if idx is None else v0[i][idx]
        return mlp.adam_update(p, g, mm, vv, k, lr)[0]

    want = [adam(0, W1, gW1), adam(1, b1, gb1), adam(2, W2, gW2), adam(3, b2, gb2)]
    rel_loss = abs(loss_g - loss_o) / loss_o
    errs = [rel_norm(after["p"][i], want[i]) for i in range(4)]
    rows = np.array(sorted(gW3_rows))
    W3_o = adam(4, W3[rows], np.stack([gW3_rows[r] for r in rows]), rows)
    b3_o = adam(5, b3[rows], np.array([gb3_rows[r] for r in rows]), rows)
    errs.append(rel_norm(after["p"][4][rows], W3_o))
    errs.append(rel_norm(after["p"][5][rows], b3_o))
    print("paper shape: loss %.6e vs %.6e (rel %.2e); tensor errs %s" % (loss_g, loss_o, rel_loss,
                                                                         ["%.1e" % e for e in errs]))
    assert rel_loss <= 2e-2
    assert max(errs) <= 1e-3
