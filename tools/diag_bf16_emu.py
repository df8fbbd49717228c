"""Diagnostic: each GPU bf16 step vs a re-anchored fp64 oracle step that applies the
same bf16 roundings (W3 shadow, H2, dY); per-tensor errors.  Differences far above
fp32 accumulation noise point at a bug."""
import os, sys
from dataclasses import replace
import numpy as np
R = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, R); sys.path.insert(0, os.path.join(R, "tests"))
from harness import FieldTable, make_config, rel_norm
from mel_inputs import design
from oracle import mlp, reservoir as ores
from paper_2309_16743_b200 import mel

def rne(x):
    return ores.bf16_bits_to_f64(ores.f32_to_bf16_bits(np.asarray(x, np.float32)))

def emu_step(p, m, v, k, S, xn, tn):
    W1, b1, W2, b2, W3, b3 = [np.asarray(x, np.float64) for x in p]
    Z1 = xn @ W1.T + b1; H1 = np.maximum(Z1, 0); Z2 = H1 @ W2.T + b2; H2 = np.maximum(Z2, 0)
    H2q, W3q = rne(H2), rne(W3)
    Y = H2q @ W3q.T + b3; Rr = Y - tn; NN = Rr.size
    loss = float(np.mean(Rr * Rr))
    g = rne(2 * Rr)                       # raw dS/dY in bf16, as K1 stores it
    gW3 = g.T @ H2q / NN; gb3 = (2 * Rr).sum(0) / NN; dH2 = g @ W3q / NN
    dZ2 = dH2 * (Z2 > 0); gW2 = dZ2.T @ H1; gb2 = dZ2.sum(0); dZ1 = (dZ2 @ W2) * (Z1 > 0)
    gW1 = dZ1.T @ xn; gb1 = dZ1.sum(0)
    lr = mlp.lr_schedule(S)
    out = [mlp.adam_update(pp, gg, mm, vv, k + 1, lr)[0] for pp, gg, mm, vv in
           zip(p, [gW1, gb1, gW2, gb2, gW3, gb3], m, v)]
    return loss, out

wl = replace(design.MEDIUM, name="medium-bf16", capacity=2000, threshold=333, sims=300)
table = FieldTable(wl)
ctx = mel.Context(make_config(wl, precision=1, storage=1))
res = ores.Reservoir(wl.capacity, wl.threshold, wl.n_field, seed=1, storage=1)
steps = 0; last = []
names = ["W1", "b1", "W2", "b2", "W3", "b3"]
for op in design.build_oplog(wl):
    if op[0] == "PUT":
        _, r, s, t = op; f = table.field(s, t); ctx.put(s, t, table.Xs(s), f); res.put(s, t, table.Xs(s), f)
    elif op[0] == "SAMPLE":
        st, last = res.sample(wl.batch); ctx.sample()
    elif op[0] == "STEP":
        if not last:
            ctx.step(); continue
        before = ctx.get_state(); st, lg = ctx.step(want_loss=True); after = ctx.get_state()
        s_ = np.asarray(last)
        xn = mlp.normalise_inputs(res.X[s_], res.t[s_], wl.tau); tn = ores.stored_to_f64(res.payload[s_], 1)
        lo, po = emu_step(before["p"], before["m"], before["v"], before["k"], before["S"], xn, tn)
        errs = [rel_norm(a, b) for a, b in zip(after["p"], po)]
        # per-tensor update error relative to the update size
        uerr = [rel_norm(np.asarray(a, np.float64) - np.asarray(b, np.float64), np.asarray(c_, np.float64) - np.asarray(b, np.float64))
                for a, b, c_ in zip(after["p"], before["p"], po)]
        steps += 1
        if steps in (1, 2, 3, 5, 10, 20, 40, 60):
            print("step %3d loss rel %.2e | weight rel %s | update rel %s" % (steps, abs(lg - lo) / lo,
                  " ".join("%s %.1e" % (n, e) for n, e in zip(names, errs)),
                  " ".join("%s %.1e" % (n, e) for n, e in zip(names, uerr))), flush=True)
        last = []
        if steps >= 60: break
