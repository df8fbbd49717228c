"""Diagnostic (not a test): per-step re-anchored errors of bf16 mode over many
steps, and free-running loss error curves for fp32 and bf16 modes."""
import os, sys
from dataclasses import replace
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from harness import FieldTable, make_config, replay_parity
from mel_inputs import design
from oracle import trainer as otr
from paper_2309_16743_b200 import mel

wl = replace(design.MEDIUM, name="medium-bf16", capacity=2000, threshold=333, sims=300)
table = FieldTable(wl)
ctx = mel.Context(make_config(wl, precision=1, storage=1))
errs = []
def on_step(ctx, res, loss, s):
    pass
rep = replay_parity(ctx, wl, table, design.build_oplog(wl), storage=1, max_train_steps=150)
le, we = np.array(rep["loss_err"]), np.array(rep["w_err"])
print("reanchored bf16: steps %d  loss err max %.2e at %d, median %.2e | w err max %.2e at %d, median %.2e" %
      (len(le), le.max(), le.argmax(), np.median(le), we.max(), we.argmax(), np.median(we)))
print("per-10 max loss err:", ["%.1e" % x for x in le.reshape(-1, 10).max(1)])
print("per-10 max w err:", ["%.1e" % x for x in we.reshape(-1, 10).max(1)])
for prec in (0, 1):
    wl2 = replace(design.MEDIUM, name="m1k", capacity=6000, threshold=1000, sims=1100)
    t2 = FieldTable(wl2)
    c2 = mel.Context(make_config(wl2, precision=prec, storage=prec))
    tr = otr.Trainer(wl2.n_field, wl2.hidden, wl2.tau, wl2.capacity, wl2.threshold, wl2.batch, seed=1, storage=prec)
    lg, lo = [], []
    for op in design.build_oplog(wl2):
        if op[0] == "PUT":
            _, r, s, t = op
            c2.put(s, t, t2.Xs(s), t2.field(s, t)); tr.put(0, s, t, t2.Xs(s), t2.field(s, t))
        elif op[0] == "SAMPLE":
            c2.sample(); tr.sample(0)
        elif op[0] == "STEP":
            a, l1 = c2.step(want_loss=True); b, l2 = tr.step()
            if a == 0:
                lg.append(l1); lo.append(l2)
                if len(lg) == 1000: break
    e = np.abs(np.array(lg) - np.array(lo)) / np.array(lo)
    print("free-running prec %d: rel loss err at steps 1,10,100,200,400,600,800,1000:" % prec,
          ["%.1e" % e[i] for i in (0, 9, 99, 199, 399, 599, 799, 999)], "mean last 50 %.2e" % e[-50:].mean())
